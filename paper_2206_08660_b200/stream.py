"""Overlapped frame stream: generate + render a sequence of volumes (one per
simulation timestep) with the host copies hidden behind the kernels.

The reference serves one frame at a time: `generate_vdi` (generate.py:444-479)
then `render_vdi` (raycast.py:459-491), host arrays in and out. On a B200 the
host link (PCIe Gen5) moves a C3 frame's 0.83 GB volume in and its 1.07 GB
of results out in about as long as the kernels take, so serialising them
nearly doubles the frame time. FrameStream runs three CUDA streams over
double-buffered HBM and pinned host slots:

    h2d     : volume i+1  host -> HBM slot (i+1) % 2
    compute : volume prep, generation, grid, (exchange,) render of frame i,
              then the results are packed into output slot i % 2 (counts,
              AoS segs, AccelGrid, image)
    d2h     : results of frame i-1  HBM slot -> pinned host slot (i-1) % 2

Every frame still performs its full H2D and D2H; only their overlap with the
neighbouring frames' kernels changes. Events order the slot reuse: an upload
waits for the compute that last read its slot, a frame's compute waits for
its upload and for the download that last read its output slot.

Results are handed out as numpy views of the pinned host slot: they stay
valid until the frame two submissions later is submitted (copy them to keep
them longer).
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
    counts: np.ndarray   # (rows, W) i32, this rank's generation rows
    segs: np.ndarray     # (rows, W, n_sg, 6) f32 AoS [front, back, r, g, b, a]
    grid: np.ndarray     # (gz, gy, gx) u32 AccelGrid counts (summed over ranks)
    image: np.ndarray    # (out_rows, out_w, 4) f64 premultiplied RGBA, this rank's rows

    @property
    def nbytes(self) -> int:
        return self.counts.nbytes + self.segs.nbytes + self.grid.nbytes + self.image.nbytes


class FrameStream:
    """Overlapped generate -> render over a stream of host volumes.

    pipe: a shard.Pipeline (N = 1 or a band-sharded rank); it owns the
    generation / render buffers and runs each frame's kernels (and, for
    N > 1, the NCCL exchange) on the compute stream.
    """

    def __init__(self, pipe):
        t = dv.require_cuda()
        self.t, self.pipe = t, pipe
        vol = pipe.vol
        shape = tuple(pipe.vol_dev.shape)
        self.h2d, self.comp, self.d2h = (t.cuda.Stream() for _ in range(3))
        self.vol_slots = [t.empty(shape, dtype=pipe.vol_dev.dtype, device="cuda")
                          for _ in range(2)]
        n_sg, w = pipe.params.n_sg, pipe.w
        rows = pipe.gen_rows
        gz, gy, gx = pipe.grid_dims[2], pipe.grid_dims[1], pipe.grid_dims[0]
        self.out = []
        self.host = []
        for _ in range(2):
            self.out.append({
                "counts": t.empty((rows, w), dtype=t.int32, device="cuda"),
                "segs": t.empty((rows * w, n_sg * 6), dtype=t.float32, device="cuda"),
                "grid": t.empty((gz, gy, gx), dtype=t.int32, device="cuda"),
                "image": t.empty(tuple(pipe.image.shape), dtype=t.float64, device="cuda"),
            })
            self.host.append({k: t.empty(v.shape, dtype=v.dtype, pin_memory=True)
                              for k, v in self.out[-1].items()})
        ev = lambda: t.cuda.Event()  # noqa: E731
        self.ev_h2d = [ev(), ev()]       # upload of slot s done
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
        voxel type, ideally pinned (dv.pinned_numpy) so the upload is async."""
        t, p = self.t, self.pipe
        i, s = self.n, self.n % 2
        src = t.from_numpy(np.ascontiguousarray(host_volume).reshape(self.vol_shape))
        with t.cuda.stream(self.h2d):
            if self.used_vol[s]:
                self.h2d.wait_event(self.ev_comp[s])
            self.vol_slots[s].copy_(src, non_blocking=True)
            self.ev_h2d[s].record(self.h2d)
        self.used_vol[s] = True
        self.h2d_bytes = src.numel() * src.element_size()
        out = self.out[s]
        with t.cuda.stream(self.comp):
            self.comp.wait_event(self.ev_h2d[s])
            if self.used_out[s]:
                self.comp.wait_event(self.ev_d2h[s])
            p.step(vol_dev=self.vol_slots[s])
            L = _capi.load()
            _capi.check(L.vdi_segs_to_aos(dv.ptr(p.bufs.segs), dv.ptr(out["segs"]),
                                          p.gen_rows * p.w, p.params.n_sg,
                                          dv.stream_handle()))
            out["counts"].copy_(p.bufs.counts, non_blocking=True)
            out["grid"].copy_(p.bufs.grid, non_blocking=True)
            out["image"].copy_(p.image, non_blocking=True)
            self.ev_comp[s].record(self.comp)
        self.used_out[s] = True
        with t.cuda.stream(self.d2h):
            self.d2h.wait_event(self.ev_comp[s])
            for k, v in out.items():
                self.host[s][k].copy_(v, non_blocking=True)
            self.ev_d2h[s].record(self.d2h)
        self.pending.append(i)
        self.n += 1

    def collect(self) -> FrameResult:
        """Wait for the oldest pending frame and return its host results."""
        i = self.pending.pop(0)
        s = i % 2
        self.ev_d2h[s].synchronize()
        h = self.host[s]
        p = self.pipe
        res = FrameResult(
            index=i,
            counts=h["counts"].numpy(),
            segs=h["segs"].numpy().reshape(p.gen_rows, p.w, p.params.n_sg, 6),
            grid=h["grid"].numpy().view(np.uint32),
            image=h["image"].numpy())
        self.d2h_bytes = res.nbytes
        return res

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
