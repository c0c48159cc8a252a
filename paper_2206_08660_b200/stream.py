"""Overlapped frame stream: generate + render a sequence of volumes (one per
simulation timestep) with the host copies hidden behind the kernels.

The reference serves one frame at a time: `generate_vdi` (generate.py:444-479)
then `render_vdi` (raycast.py:459-491), host arrays in and out. On a B200 the
host link (PCIe Gen5) moves a C3 frame's 0.83 GB volume in and its 1.07 GB
of results out in about as long as the kernels take, so serialising them
nearly doubles the frame time. FrameStream runs three CUDA streams over
double-buffered HBM and pinned host slots:

    h2d     : volume i+1  host -> HBM slot (i+1) % 2
    compute : volume prep, generation, grid of frame i
    render  : render of frame i, then the results are packed into output
              slot i % 2 (counts, AoS segs or VDI1 bytes, AccelGrid, image)
    d2h     : results of frame i-1  HBM slot -> pinned host slot (i-1) % 2

With one rank the render of frame i runs on its own stream, beside the
volume prep of frame i+1 (which reads neither the VDI nor the image); the
generation of frame i+1 waits for it (one set of generation buffers). With
N > 1 ranks the whole step, collectives included, stays on the compute
stream.

Every frame still performs its full H2D and D2H; only their overlap with the
neighbouring frames' kernels changes. Events order the slot reuse: an upload
waits for the compute that last read its slot, a frame's compute waits for
its upload and for the download that last read its output slot.

At most two frames are in flight: `submit` raises if two submitted frames
have not been collected yet. Results are handed out as numpy views of the
pinned host slot: they stay valid until the frame two submissions later is
submitted (its readback reuses the slot; copy them to keep them longer). In
packed mode frame i's VDI1 bytes are copied to the host inside collect(i),
which the in-flight limit orders before submit(i + 2) re-encodes the slot.

packed=True returns the VDI in the reference's own wire/file format instead
of the dense (H, W, n_sg, 6) array: the VDI1 byte string of
`encode_vdi(vdi, grid)` (vdi.py:141-159, bit-identical; `decode_vdi` rebuilds
the identical Vdi and AccelGrid), packed on the device (vdi_encode_vdi1).
Only valid supersegments cross the host link (C3: 183 MB instead of 1 GB).
The packed length is known on the device only, so a frame's length and image
are read back on the d2h stream with the frame, and its VDI1 bytes are
copied once `collect` has read the length -- still overlapped with the next
frame's kernels, which are queued by then.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _capi
from . import device as dv


@dataclass
class FrameResult:
    """Host results of one frame (views of a pinned slot; see module doc)."""
    index: int
    counts: np.ndarray | None  # (rows, W) i32, this rank's generation rows
    segs: np.ndarray | None    # (rows, W, n_sg, 6) f32 AoS [front, back, r, g, b, a]
    grid: np.ndarray | None    # (gz, gy, gx) u32 AccelGrid counts (summed over ranks)
    image: np.ndarray          # (out_rows, out_w, 4) f64 premultiplied RGBA, this rank's rows
    vdi1: np.ndarray | None = None  # packed mode: the VDI1 bytes (u8)

    @property
    def nbytes(self) -> int:
        if self.vdi1 is not None:
            return self.vdi1.nbytes + self.image.nbytes + 8
        return self.counts.nbytes + self.segs.nbytes + self.grid.nbytes + self.image.nbytes

    def decode(self):
        """(counts, segs, grid) from the VDI1 bytes (vdi.py:162-210 layout)."""
        if self.vdi1 is None:
            return self.counts, self.segs, self.grid
        import struct
        b = self.vdi1
        _, _, w, h, n_sg = struct.unpack_from("<4sIIII", b, 0)
        gx, gy, gz = struct.unpack_from("<3I", b, 148)
        off = 160
        counts = np.frombuffer(b, "<u2", w * h, off).reshape(h, w).astype(np.int32)
        off += 2 * w * h
        total = int(counts.sum())
        packed = np.frombuffer(b, "<f4", 6 * total, off).reshape(total, 6)
        off += 24 * total
        grid = np.frombuffer(b, "<u4", gx * gy * gz, off).reshape(gz, gy, gx)
        segs = np.zeros((h, w, n_sg, 6), np.float32)
        segs[np.arange(n_sg)[None, None, :] < counts[:, :, None]] = packed
        return counts, segs, grid


class FrameStream:
    """Overlapped generate -> render over a stream of host volumes.

    pipe: a shard.Pipeline (N = 1 or a band-sharded rank); it owns the
    generation / render buffers and runs each frame's kernels (and, for
    N > 1, the NCCL exchange) on the compute stream.
    """

    def __init__(self, pipe, packed: bool = False):
        t = dv.require_cuda()
        if getattr(pipe, "bricked", False):
            raise NotImplementedError("FrameStream: a bricked pipeline keeps only its voxel "
                                      "box resident; whole-volume frames do not fit it")
        self.t, self.pipe, self.packed = t, pipe, packed
        vol = pipe.vol
        shape = tuple(pipe.vol_dev.shape)
        self.h2d, self.comp, self.d2h = (t.cuda.Stream() for _ in range(3))
        # one rank: the render and the packing of frame i beside frame i+1's prep
        self.split = getattr(pipe, "world", 1) == 1
        self.rend = t.cuda.Stream() if self.split else self.comp
        # packed mode: the variable-length VDI1 copy gets its own stream, so it
        # does not queue behind the next frame's fixed-size readback (which
        # waits for that frame's kernels)
        self.d2h_var = t.cuda.Stream()
        self.ev_var = t.cuda.Event()
        self.vol_slots = [t.empty(shape, dtype=pipe.vol_dev.dtype, device="cuda")
                          for _ in range(2)]
        n_sg, w = pipe.params.n_sg, pipe.w
        rows = pipe.gen_rows
        gz, gy, gx = pipe.grid_dims[2], pipe.grid_dims[1], pipe.grid_dims[0]
        self.out = []
        self.host = []
        L = _capi.load()
        self.vdi1_cap = int(L.vdi_vdi1_max_bytes(w, rows, n_sg, gx, gy, gz))
        self.enc_ws = t.empty(int(L.vdi_encode_workspace_bytes(w, rows)), dtype=t.uint8,
                              device="cuda")
        for _ in range(2):
            if packed:
                o = {"vdi1": t.empty(self.vdi1_cap, dtype=t.uint8, device="cuda"),
                     "len": t.zeros(1, dtype=t.int64, device="cuda"),
                     "image": t.empty(tuple(pipe.image.shape), dtype=t.float64,
                                      device="cuda")}
            else:
                o = {"counts": t.empty((rows, w), dtype=t.int32, device="cuda"),
                     "segs": t.empty((rows * w, n_sg * 6), dtype=t.float32, device="cuda"),
                     "grid": t.empty((gz, gy, gx), dtype=t.int32, device="cuda"),
                     "image": t.empty(tuple(pipe.image.shape), dtype=t.float64,
                                      device="cuda")}
            self.out.append(o)
            self.host.append({k: t.empty(v.shape, dtype=v.dtype, pin_memory=True)
                              for k, v in o.items()})
        ev = lambda: t.cuda.Event()  # noqa: E731
        self.ev_h2d = [ev(), ev()]       # upload of slot s done
        self.ev_vol = [ev(), ev()]       # the kernels that read vol slot s are done
        self.ev_gen = ev()               # the last frame's generation is done
        self.ev_rend = ev()              # the last frame's render / packing is done
        self.ev_comp = [ev(), ev()]      # compute that read vol slot / wrote out slot s done
        self.ev_d2h = [ev(), ev()]       # download of out slot s done
        self.used_vol = [False, False]
        self.used_out = [False, False]
        self.pending = []                # frame indices submitted, not yet collected
        self.n = 0
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.vol_shape = (vol.dims[2], vol.dims[1], vol.dims[0])

    def submit(self, host_volume: np.ndarray) -> None:
        """Queue one frame. host_volume: (nz, ny, nx) array of the pipeline's
        voxel type, ideally pinned (dv.pinned_numpy) so the upload is async.
        Raises RuntimeError when two frames are already in flight (collect
        the oldest first: their slots would be overwritten)."""
        if len(self.pending) >= 2:
            raise RuntimeError("FrameStream: two frames in flight; collect() the oldest first")
        t, p = self.t, self.pipe
        i, s = self.n, self.n % 2
        src = t.from_numpy(np.ascontiguousarray(host_volume).reshape(self.vol_shape))
        with t.cuda.stream(self.h2d):
            if self.used_vol[s]:
                self.h2d.wait_event(self.ev_vol[s])
            self.vol_slots[s].copy_(src, non_blocking=True)
            self.ev_h2d[s].record(self.h2d)
        self.used_vol[s] = True
        self.h2d_bytes = src.numel() * src.element_size()
        out = self.out[s]
        with t.cuda.stream(self.comp):
            self.comp.wait_event(self.ev_h2d[s])
            if self.split:
                p.prep(self.vol_slots[s])
                # the generation rewrites the VDI the previous render reads
                self.comp.wait_event(self.ev_rend)
                p.launch_gen(self.vol_slots[s])
                self.ev_gen.record(self.comp)
            else:
                if self.used_out[s]:
                    self.comp.wait_event(self.ev_d2h[s])
                p.step(vol_dev=self.vol_slots[s])
            self.ev_vol[s].record(self.comp)
        with t.cuda.stream(self.rend):
            if self.split:
                self.rend.wait_event(self.ev_gen)
                if self.used_out[s]:
                    self.rend.wait_event(self.ev_d2h[s])
                p.launch_render()
            L = _capi.load()
            if self.packed:
                _capi.check(L.vdi_encode_vdi1(self._enc_args(out), dv.stream_handle()))
            else:
                _capi.check(L.vdi_segs_to_aos(dv.ptr(p.bufs.segs), dv.ptr(out["segs"]),
                                              p.gen_rows * p.w, p.params.n_sg,
                                              dv.stream_handle()))
                out["counts"].copy_(p.bufs.counts, non_blocking=True)
                out["grid"].copy_(p.bufs.grid, non_blocking=True)
            out["image"].copy_(p.image, non_blocking=True)
            self.ev_comp[s].record(self.rend)
            self.ev_rend.record(self.rend)
        self.used_out[s] = True
        with t.cuda.stream(self.d2h):
            self.d2h.wait_event(self.ev_comp[s])
            for k, v in out.items():
                if k != "vdi1":  # packed: its length is read first (collect)
                    self.host[s][k].copy_(v, non_blocking=True)
            self.ev_d2h[s].record(self.d2h)
        self.pending.append(i)
        self.n += 1

    def collect(self) -> FrameResult:
        """Wait for the oldest pending frame and return its host results."""
        if not self.pending:
            raise RuntimeError("FrameStream: no frame in flight")
        i = self.pending.pop(0)
        s = i % 2
        self.ev_d2h[s].synchronize()
        h = self.host[s]
        p = self.pipe
        if self.packed:
            n = int(h["len"][0])
            with self.t.cuda.stream(self.d2h_var):
                self.d2h_var.wait_event(self.ev_comp[s])
                h["vdi1"][:n].copy_(self.out[s]["vdi1"][:n], non_blocking=True)
                self.ev_var.record(self.d2h_var)
                self.ev_d2h[s].record(self.d2h_var)  # slot s is free after this copy
            self.ev_var.synchronize()
            res = FrameResult(index=i, counts=None, segs=None, grid=None,
                              image=h["image"].numpy(), vdi1=h["vdi1"][:n].numpy())
            self.d2h_bytes = res.nbytes
            return res
        res = FrameResult(
            index=i,
            counts=h["counts"].numpy(),
            segs=h["segs"].numpy().reshape(p.gen_rows, p.w, p.params.n_sg, 6),
            grid=h["grid"].numpy().view(np.uint32),
            image=h["image"].numpy())
        self.d2h_bytes = res.nbytes
        return res

    def _enc_args(self, out):
        """vdi_encode_vdi1 arguments for this rank's generation rows."""
        from .codec import vdi1_header
        from .vdi import AccelGrid, Vdi
        p = self.pipe
        if not hasattr(self, "_hdr"):
            vdi = Vdi(p.w, p.gen_rows, p.params.n_sg, None, None, p.gcam, p.aabb)
            self._hdr = vdi1_header(vdi, AccelGrid(p.grid_dims, None, p.gcam.near, p.gcam.far))
        a = _capi.VdiEncodeArgs()
        a.segs, a.counts, a.grid = dv.ptr(p.bufs.segs), dv.ptr(p.bufs.counts), dv.ptr(p.bufs.grid)
        a.out, a.out_len = dv.ptr(out["vdi1"]), dv.ptr(out["len"])
        a.workspace, a.workspace_bytes = dv.ptr(self.enc_ws), int(self.enc_ws.numel())
        for k, b in enumerate(self._hdr):
            a.header[k] = b
        a.width, a.height, a.n_sg = p.w, p.gen_rows, p.params.n_sg
        a.gx, a.gy, a.gz = (int(v) for v in p.grid_dims)
        a.vdi_band_rows, a.vdi_band_world, a.vdi_rows_per_rank = 16, 1, p.gen_rows
        return a

    def run(self, volumes, on_result=None):
        """Submit every volume, collecting each frame once the next one is
        queued (so two frames are in flight); returns the number of frames."""
        n = 0
        for vol in volumes:
            self.submit(vol)
            if len(self.pending) > 1:
                r = self.collect()
                if on_result is not None:
                    on_result(r)
            n += 1
        while self.pending:
            r = self.collect()
            if on_result is not None:
                on_result(r)
        return n
