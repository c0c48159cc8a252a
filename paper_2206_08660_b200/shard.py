"""Ray-band sharding of generate -> render across the GPUs of one box.

Both passes are independent per ray (generate.py:281 / raycast.py:283
`prange`), so each rank takes the interleaved 16-row bands b with
b % world == rank of the generation viewport and of the output viewport
(interleaving balances empty borders and 1- vs 22-pass rays). The only
exchange is between the passes: the render rays of any rank can traverse any
list, so the AccelGrid partials are all-reduced (sum) and the VDI tiles are
all-gathered (NCCL over NVLink); the gathered VDI is read in its
band-interleaved storage order through the band map (include/vdi_b200.h), so
no permutation copy is made. The image rows are all-gathered at the end.

The collectives go through torch.distributed, so the same host logic runs
with NCCL on B200s and with gloo on CPU tensors in the tests.
"""

from __future__ import annotations

import time
import weakref

import numpy as np

from . import _capi
from . import device as dv
from .generate import alloc_gen, launch_generate
from .raycast import (RenderOptions, alloc_list_tiles, alloc_ranges, alloc_tile_counter,
                      alloc_zmask, launch_list_tiles, launch_ranges, launch_zmask, render_args,
                      set_tile_counter, use_list_ranges, use_list_tiles)
from .vdi import AccelGrid, DeviceVdi, Vdi, default_grid_dims

BAND_ROWS = 16


def band_rows(height: int, world: int, rank: int, band: int = BAND_ROWS) -> np.ndarray:
    """Image rows owned by `rank` (same rule as band_global_row in the kernels)."""
    rows = np.arange(height)
    return rows[(rows // band) % world == rank]


def local_rows(height: int, world: int, rank: int, band: int = BAND_ROWS) -> int:
    return int(len(band_rows(height, world, rank, band)))


def rows_per_rank(height: int, world: int, band: int = BAND_ROWS) -> int:
    """Padded per-rank row count (rank 0 owns the most rows)."""
    return local_rows(height, world, 0, band)


def storage_rows(height: int, world: int, band: int = BAND_ROWS) -> np.ndarray:
    """Storage row of each image row after an all-gather of padded shards
    (vdi_storage_row in the kernels)."""
    if world <= 1:
        return np.arange(height)
    r = np.arange(height)
    b = r // band
    return (b % world) * rows_per_rank(height, world, band) + (b // world) * band + r % band


def gather_rows(dist, local, world: int, padded_rows: int):
    """All-gather equal-size (padded) row shards: [world * padded_rows, ...]."""
    if local.shape[0] != padded_rows:
        raise ValueError("shard must be padded to rows_per_rank rows")
    out = local.new_empty((world * padded_rows, *local.shape[1:]))
    dist.all_gather_into_tensor(out, local.contiguous())
    return out


def band_volume_box(vol, cam, row0: int, row1: int, margin: int = 2, align: int = 8):
    """Voxel box (origin, size) holding every cell the generation rays of
    image rows [row0, row1) can sample: the rays' clipped chords
    (generate.py:282-306, evaluated for every pixel of the band, f64 as the
    kernels do) -> normalised positions -> trilinear cells (+1 neighbour),
    widened by `margin` voxels for rounding and aligned to the brick edge.
    With an elevation-0 orbit camera a contiguous row band maps to a y-slab
    of the volume (SURVEY.md 8(e), C5 "bricked across 8")."""
    w, h = cam.viewport
    dims = np.array(vol.dims, np.int64)
    lo_b, hi_b = np.asarray(vol.aabb, np.float64)
    inv = np.asarray(cam.inv_proj_view(), np.float64)
    pv = np.asarray(cam.proj_view(), np.float64)
    eye = np.asarray(cam.position, np.float64)
    cols = np.arange(w)
    rows = np.arange(row0, row1)
    X, Y = np.meshgrid(2.0 * (cols + 0.5) / w - 1.0, 2.0 * (rows + 0.5) / h - 1.0)
    P = np.stack([X.ravel(), Y.ravel(), -np.ones(X.size), np.ones(X.size)], 1) @ inv.T
    P = P[:, :3] / P[:, 3:4]
    D = P - eye
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    with np.errstate(divide="ignore", invalid="ignore"):
        ta = (lo_b - eye) / D
        tb = (hi_b - eye) / D
    t0 = np.nanmax(np.minimum(ta, tb), axis=1)
    t1 = np.nanmin(np.maximum(ta, tb), axis=1)
    # generation frustum (7 half-spaces c + t d >= 0), as clip_frustum
    c4 = np.append(eye, 1.0) @ pv.T
    d4 = np.concatenate([D, np.zeros((len(D), 1))], 1) @ pv.T
    cs = np.stack([c4[3], c4[3] - c4[0], c4[3] + c4[0], c4[3] - c4[1], c4[3] + c4[1],
                   c4[3] - c4[2], c4[3] + c4[2]])
    ds = np.stack([d4[:, 3], d4[:, 3] - d4[:, 0], d4[:, 3] + d4[:, 0], d4[:, 3] - d4[:, 1],
                   d4[:, 3] + d4[:, 1], d4[:, 3] - d4[:, 2], d4[:, 3] + d4[:, 2]], 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        tt = -cs[None, :] / ds
    fa = np.max(np.where(ds > 0, tt, -np.inf), axis=1)
    fb = np.min(np.where(ds < 0, tt, np.inf), axis=1)
    t0 = np.maximum(np.maximum(t0, fa), 0.0)
    t1 = np.minimum(t1, fb)
    hit = t1 > t0
    if not hit.any():
        return (0, 0, 0), (min(int(dims[0]), align), min(int(dims[1]), align),
                           min(int(dims[2]), align))
    ends = np.concatenate([eye + t0[hit, None] * D[hit], eye + t1[hit, None] * D[hit]])
    q = np.clip((ends - lo_b) / (hi_b - lo_b), 0.0, 1.0) * (dims - 1)
    cmin = np.floor(q.min(0)).astype(np.int64) - margin
    cmax = np.floor(q.max(0)).astype(np.int64) + 1 + margin
    org = np.clip((cmin // align) * align, 0, None)
    end = np.minimum(cmax + 1, dims)
    return tuple(int(v) for v in org), tuple(int(v) for v in end - org)


def brick_slabs(nz: int, world: int, log2: int = 3):
    """Brick z-planes per rank for the sharded brick maxima: rank r computes
    planes [r P, min((r + 1) P, nbz)) with P = ceil(nbz / world), from voxel
    planes [8 r P, min(8 (r + 1) P + 1, nz)) (the +1: a brick's trilinear
    halo). Returns (P, nbz, [(z0, z1, planes)] per rank)."""
    b = 1 << log2
    nbz = -(-nz // b)
    per = -(-nbz // world)
    out = []
    for r in range(world):
        p0, p1 = min(r * per, nbz), min((r + 1) * per, nbz)
        z0, z1 = p0 * b, min(p1 * b + 1, nz)
        out.append((z0, z1, p1 - p0))
    return per, nbz, out


def balance_bands(row_cost, world: int) -> list:
    """Boundaries b_0 = 0 < ... < b_world = H of contiguous row bands with
    near-equal total cost (row_cost: per-image-row work, e.g. the executed
    samples of the previous frame's rows): b_r is the first row whose cost
    prefix reaches r / world of the total. Every band keeps >= 1 row."""
    c = np.asarray(row_cost, np.float64)
    h = len(c)
    pre = np.concatenate([[0.0], np.cumsum(np.maximum(c, 0.0) + 1e-9)])
    tot = pre[-1]
    b = [0]
    for r in range(1, world):
        k = int(np.searchsorted(pre, tot * r / world, side="left"))
        b.append(min(max(k, b[-1] + 1), h - (world - r)))
    b.append(h)
    return b


def row_storage_map(bounds, rows_per_rank: int) -> np.ndarray:
    """Storage row of every image row after the all-gather of contiguous
    bands padded to rows_per_rank (VdiRenderArgs.vdi_row_map)."""
    out = np.empty(bounds[-1], np.int32)
    for q in range(len(bounds) - 1):
        r0, r1 = bounds[q], bounds[q + 1]
        out[r0:r1] = q * rows_per_rank + np.arange(r1 - r0)
    return out


class PackedExchange:
    """The VDI exchange as packed VDI1 shards instead of the padded list-SoA:
    each rank packs its rows (vdi_encode_vdi1: counts u16 + valid
    supersegments only, 183 MB instead of 995 MB for a whole C3 frame), the
    ranks all-gather the lengths and the packed shards (padded to the
    longest), and every rank unpacks all shards into the band-interleaved
    list-SoA storage the render kernel reads (vdi_decode_vdi1_lists). The
    AccelGrid partials are still all-reduced. Bit-identical to exchange_vdi."""

    def __init__(self, pipe):
        t = dv.torch()
        L = _capi.load()
        # a proxy, not a reference: Pipeline owns this object, and a cycle
        # would keep its (tens of GB of) device buffers alive after `del`
        self.pipe = weakref.proxy(pipe)
        w, rows, n_sg = pipe.w, pipe.gen_rows, pipe.params.n_sg
        self.cap = int(L.vdi_vdi1_max_bytes(w, rows, n_sg, 1, 1, 1))
        self.buf = t.zeros(self.cap, dtype=t.uint8, device="cuda")
        self.len = t.zeros(1, dtype=t.int64, device="cuda")
        self.lens = t.zeros(pipe.world, dtype=t.int64, device="cuda")
        ws = int(L.vdi_encode_workspace_bytes(w, rows))
        self.enc_ws = t.empty(ws, dtype=t.uint8, device="cuda")
        self.dec_ws = t.empty(ws, dtype=t.uint8, device="cuda")
        self.dummy_grid = t.zeros(1, dtype=t.int32, device="cuda")
        # the gather buffer at full capacity, allocated once (each frame
        # gathers world x max(lens) bytes into its head)
        self.g_buf = t.empty(pipe.world * self.cap, dtype=t.uint8, device="cuda")
        a = _capi.VdiEncodeArgs()
        a.segs, a.counts, a.grid = (dv.ptr(pipe.bufs.segs), dv.ptr(pipe.bufs.counts),
                                    dv.ptr(self.dummy_grid))
        a.out, a.out_len = dv.ptr(self.buf), dv.ptr(self.len)
        a.workspace, a.workspace_bytes = dv.ptr(self.enc_ws), ws
        hdr = np.zeros(_capi.VDI1_HEADER_BYTES, np.uint8)  # unused by the receiver
        for k, b in enumerate(hdr.tobytes()):
            a.header[k] = b
        a.width, a.height, a.n_sg = w, rows, n_sg
        a.gx = a.gy = a.gz = 1
        a.vdi_band_rows, a.vdi_band_world, a.vdi_rows_per_rank = 16, 1, rows
        self.args = a
        self.bytes_last = 0

    def __call__(self, dist, grid, g_counts, g_segs):
        L = _capi.load()
        p = self.pipe
        dist.all_reduce(grid)
        _capi.check(L.vdi_encode_vdi1(self.args, dv.stream_handle()))
        dist.all_gather_into_tensor(self.lens, self.len)
        # the gather is sized by the longest shard: one 8-byte-per-rank host
        # read (NCCL sizes are host values). exchange_vdi is the sync-free
        # alternative (the padded list-SoA, 5.4x the bytes at C3).
        lens = self.lens.cpu().tolist()
        m = int(max(lens))
        g_buf = self.g_buf[:p.world * m]
        dist.all_gather_into_tensor(g_buf, self.buf[:m])
        w, rows, n_sg = p.w, p.gen_rows, p.params.n_sg
        stride = g_segs.shape[1]
        for q in range(p.world):
            src = g_buf[q * m:(q + 1) * m]
            cq = g_counts[q * rows:(q + 1) * rows]
            sq = g_segs[q * rows * w:(q + 1) * rows * w]
            _capi.check(L.vdi_decode_vdi1_lists(dv.ptr(src), w, rows, n_sg, dv.ptr(cq),
                                                dv.ptr(sq), dv.ptr(self.dec_ws),
                                                int(self.dec_ws.numel()), dv.stream_handle()))
        assert stride == list_stride_of(n_sg)
        self.bytes_last = int(sum(lens))


def list_stride_of(n_sg: int) -> int:
    return (6 * n_sg + 3) & ~3


def exchange_vdi(dist, counts, segs, grid, g_counts, g_segs):
    """The one exchange between generation and rendering: sum the partial
    AccelGrids in place and all-gather the padded VDI shards (counts
    [rows, W], segs [rows * W, stride]) into band-interleaved storage."""
    dist.all_reduce(grid)
    dist.all_gather_into_tensor(g_counts, counts)
    dist.all_gather_into_tensor(g_segs, segs)


class Pipeline:
    """generate -> (all-reduce grid, all-gather VDI) -> render -> all-gather
    image, device-resident, for one rank."""

    def __init__(self, vol, tf, gcam, rcam, params, world=1, rank=0, opts=None,
                 bricked=False, box_volume=None, band_bounds=None):
        """bricked: generation takes contiguous row bands (rank r: rows
        [r B, (r + 1) B), B = ceil(H / world)) and keeps only the voxel box
        those rays sample (band_volume_box) resident -- the C5 placement,
        "bricked across 8 x B200". box_volume(origin, size) -> device tensor
        (size[2], size[1], size[0]) supplies that box (default: sliced from
        `vol`). band_bounds (bricked): world + 1 row boundaries of contiguous
        bands of unequal height (balance_bands of the previous frame's
        per-row cost) instead of equal ones. Rendering keeps the interleaved
        16-row bands."""
        t = dv.require_cuda()
        self.t = t
        self.vol, self.tf, self.gcam, self.rcam, self.params = vol, tf, gcam, rcam, params
        self.world, self.rank = world, rank
        self.opts = opts or RenderOptions()
        self.resolved = params.resolve(vol)
        w, h = gcam.viewport
        self.w, self.h = w, h
        self.grid_dims = default_grid_dims(w, h)
        self.bricked = bricked
        self.gen_band_rows = -(-h // world) if bricked else BAND_ROWS
        self.sub = None
        self.gen_range = None  # (row_base, row_count) of unequal contiguous bands
        self.band_bounds = None
        if bricked and band_bounds is not None:
            self.band_bounds = [int(x) for x in band_bounds]
            assert len(self.band_bounds) == world + 1 and self.band_bounds[-1] == h
        if bricked:
            if self.band_bounds is not None:
                r0, r1 = self.band_bounds[rank], self.band_bounds[rank + 1]
                self.gen_range = (r0, r1 - r0)
            else:
                r0 = rank * self.gen_band_rows
                r1 = min(h, r0 + self.gen_band_rows)
            org, size = band_volume_box(vol, gcam, r0, max(r1, r0 + 1))
            self.box = (org, size)
            if box_volume is not None:
                self.vol_dev = box_volume(org, size)
            else:
                full, _ = dv.upload_volume(vol, cache=False)
                ox, oy, oz = org
                sx, sy, sz = size
                self.vol_dev = full[oz:oz + sz, oy:oy + sy, ox:ox + sx].contiguous()
                del full
            self.vt = vol.voxel_type
            self.oob = t.zeros(1, dtype=t.int32, device="cuda")
            self.sub = (org, size, self.oob)
            self.res_dims = size
        else:
            self.box = None
            self.vol_dev, self.vt = dv.upload_volume(vol)
            self.res_dims = tuple(vol.dims)
        self.lut_dev = dv.upload_lut(tf.lut)
        # per-volume acceleration data, rebuilt from the volume inside every
        # step (a new timestep's volume needs new ones): brick maxima for
        # empty-space skipping and, when they fit, the corner records
        self.bricks = dv.alloc_bricks(self.vol_dev, self.res_dims)
        # corner records save ~8 % of a full generation but cost a full-volume
        # pass on every rank; with more than two ranks sharing the rays they
        # cost more than they save (C3: 0.93 ms vs 2.5 ms / N), so only N <= 2
        # builds them
        from .tuning import TUNING
        self.cells = (dv.alloc_cells(self.vt, self.res_dims)
                      if dv.use_cells(self.vt, self.res_dims)
                      and (world <= TUNING.cells_max_world) else None)
        # N > 1 (replicated volume): each rank computes a z-slab of the brick
        # maxima and the ranks all-gather them (1.6 MB at C3)
        self.slabs = None
        if world > 1 and not bricked:
            per, nbz, plan = brick_slabs(int(vol.dims[2]), world, dv.BRICK_LOG2)
            nby, nbx = self.bricks.shape[1], self.bricks.shape[2]
            self.bricks_all = t.empty((world * per, nby, nbx), dtype=self.bricks.dtype,
                                      device="cuda")
            self.bricks = self.bricks_all[:nbz]
            z0, z1, planes = plan[rank]
            self.slab_local = t.zeros((per, nby, nbx), dtype=self.bricks.dtype, device="cuda")
            self.slab_tmp = (t.empty((-(-(z1 - z0) // (1 << dv.BRICK_LOG2)), nby, nbx),
                                     dtype=self.bricks.dtype, device="cuda")
                             if z1 > z0 else None)
            self.slabs = (z0, z1, planes)
        self.ess_max = dv.ess_threshold(tf.lut)
        self.aabb = np.asarray(vol.aabb, np.float64)
        self.band = (BAND_ROWS, world, rank)
        self.gen_band = (self.gen_band_rows, world, rank)
        self.gen_rows = rows_per_rank(h, world, self.gen_band_rows)
        self.local_gen_rays = local_rows(h, world, rank, self.gen_band_rows) * w
        if self.gen_range is not None:
            b = self.band_bounds
            self.gen_rows = max(b[q + 1] - b[q] for q in range(world))
            self.local_gen_rays = self.gen_range[1] * w
        self.bufs = alloc_gen(w, self.gen_rows, params.n_sg, self.grid_dims, stats=True)
        self.bufs.counts.zero_()  # padding rows stay empty
        ow, oh = rcam.viewport
        self.ow, self.oh = ow, oh
        self.out_rows = rows_per_rank(oh, world)
        self.local_render_pixels = local_rows(oh, world, rank) * ow
        self.image = t.zeros((self.out_rows, ow, 4), dtype=t.float64, device="cuda")
        self.sums = t.zeros(3, dtype=t.int64, device="cuda")
        # brick maxima (+ corner records); vdi_gen_launch = fill_inv + 3 rounds
        # x (sample, fill, bisect, emit) + fused fallback; then
        # vdi_grid_launch and vdi_render_launch
        self.tiles = (alloc_list_tiles(w, h) if use_list_tiles() else None)
        self.zmask = alloc_zmask(self.grid_dims) if self.opts.use_ess else None
        # this package's kernels per step: brick maxima (+ corner records);
        # vdi_gen_launch = fill_inv + ray setup + 3 rounds x (sample, queue
        # count / scan / write, fill, bisect, wide bisect, emit) + the fused
        # fallback; grid; the render's slab words (+ tile bitmap, + list
        # ranges) and the render
        self.launches_per_step = (1 + (self.cells is not None) + 2 + 3 * 8 + 1 + 1
                                  + (self.tiles is not None) + (self.zmask is not None) + 1)
        if world > 1:
            import torch.distributed as tdist
            self.dist = tdist
            self.g_counts = t.empty((world * self.gen_rows, w), dtype=t.int32, device="cuda")
            self.g_segs = t.empty((world * self.gen_rows * w, self.bufs.segs.shape[1]),
                                  dtype=t.float32, device="cuda")
            self.g_image = t.empty((world * self.out_rows, ow, 4), dtype=t.float64,
                                   device="cuda")
            row_map = None
            if self.gen_range is not None:
                row_map = dv.to_device(row_storage_map(self.band_bounds, self.gen_rows))
            self.dvdi = DeviceVdi(self.g_counts, self.g_segs, self.gen_band_rows, world,
                                  self.gen_rows, sorted=True, row_map=row_map)
            from .tuning import TUNING
            self.packed = PackedExchange(self) if TUNING.packed_exchange else None
        else:
            self.dist = None
            self.dvdi = DeviceVdi(self.bufs.counts, self.bufs.segs, sorted=True)
        # the frame's render counts lists visited / supersegments intersected
        # (R's RenderStats) but not lists searched (search-first shading,
        # VdiRenderArgs.lists_sorted); exact_render_stats() counts all three
        self._rargs = render_args(self.dvdi, params.n_sg, w, h, gcam, self.aabb, self.bufs.grid,
                                  self.grid_dims, gcam.near, gcam.far, rcam, self.opts,
                                  self.image, stat_sums=self.sums, band=self.band,
                                  counters_exact=False)
        # per-list depth ranges of the exchanged VDI (search-first shading)
        self.n_lists = int(self.dvdi.counts.numel())
        self.ranges = alloc_ranges(self.n_lists) if use_list_ranges(self._rargs) else None
        self.launches_per_step += self.ranges is not None
        self.tile_counter = alloc_tile_counter()
        set_tile_counter(self._rargs, self.tile_counter)

    def step(self, timed: bool = False, vol_dev=None):
        """One frame on the current stream: volume prep, generation, grid,
        (exchange,) render. vol_dev: the frame's device volume (default: the
        pipeline's own copy)."""
        t = self.t
        vol_dev = self.vol_dev if vol_dev is None else vol_dev
        ev = [t.cuda.Event(enable_timing=True) for _ in range(6)] if timed else None
        if timed:
            ev[0].record()
        self.sums.zero_()
        self.prep(vol_dev)
        self.launch_gen(vol_dev, split_events=ev)
        if timed:
            ev[3].record()
        if self.world > 1:
            if self.packed is not None:
                self.packed(self.dist, self.bufs.grid, self.g_counts, self.g_segs)
            else:
                exchange_vdi(self.dist, self.bufs.counts, self.bufs.segs, self.bufs.grid,
                             self.g_counts, self.g_segs)
        if timed:
            ev[4].record()
        self.launch_render(zero_sums=False)
        if timed:
            ev[5].record()
        if self.world > 1:
            self.dist.all_gather_into_tensor(self.g_image, self.image)
        if not timed:
            return None
        end = t.cuda.Event(enable_timing=True)
        end.record()
        end.synchronize()
        return {"step": ev[0].elapsed_time(end), "prep": ev[0].elapsed_time(ev[1]),
                "gen": ev[1].elapsed_time(ev[2]),
                "grid": ev[2].elapsed_time(ev[3]),
                "collective": ev[3].elapsed_time(ev[4]) + ev[5].elapsed_time(end),
                "render": ev[4].elapsed_time(ev[5])}

    def launch_gen(self, vol_dev, split_events=None):
        """This rank's generation + partial AccelGrid of `vol_dev` (prep done),
        on the current stream."""
        launch_generate(vol_dev, self.vt, self.vol.dims, self.lut_dev, self.gcam,
                        self.aabb, self.params, self.resolved, self.bufs, self.grid_dims,
                        band=self.gen_band, split_events=split_events, bricks=self.bricks,
                        ess_max=self.ess_max, cells=self.cells, sub=self.sub,
                        rows=self.gen_range)

    def launch_render(self, zero_sums: bool = True):
        """This rank's render of the exchanged VDI into self.image (slab words,
        list ranges, render), on the current stream."""
        if zero_sums:
            self.sums.zero_()
        if self.tiles is not None:
            launch_list_tiles(self._rargs, self.tiles)
        launch_zmask(self._rargs, self.zmask)
        launch_ranges(self._rargs, self.ranges, self.n_lists)
        _capi.check(_capi.load().vdi_render_launch(self._rargs, dv.stream_handle()))

    def prep(self, vol_dev, gather: bool = True):
        """Per-volume acceleration data: brick maxima (sharded by z-slab and
        all-gathered when N > 1 with a replicated volume) and, for N <= 2,
        the corner records. gather=False leaves the other ranks' slabs as
        they are (one-GPU timing of a rank's share)."""
        if self.slabs is None:
            dv.launch_bricks(vol_dev, self.vt, self.res_dims, self.bricks)
        else:
            z0, z1, planes = self.slabs
            nx, ny = int(self.res_dims[0]), int(self.res_dims[1])
            if planes > 0:
                dv.launch_bricks(vol_dev[z0:z1], self.vt, (nx, ny, z1 - z0), self.slab_tmp)
                self.slab_local[:planes].copy_(self.slab_tmp[:planes])
            if gather:
                self.dist.all_gather_into_tensor(self.bricks_all, self.slab_local)
        if self.cells is not None:
            dv.launch_cells(vol_dev, self.vt, self.res_dims, self.cells, self.bricks, self.ess_max)

    def exact_render_stats(self):
        """(lists visited, supersegments intersected, lists searched) of this
        rank's render in the reference's ESS-then-search order (an extra,
        untimed render)."""
        t = self.t
        sums = t.zeros(3, dtype=t.int64, device="cuda")
        a = render_args(self.dvdi, self.params.n_sg, self.w, self.h, self.gcam, self.aabb,
                        self.bufs.grid, self.grid_dims, self.gcam.near, self.gcam.far,
                        self.rcam, self.opts, self.image, stat_sums=sums, band=self.band,
                        counters_exact=True)
        launch_zmask(a, self.zmask)
        set_tile_counter(a, self.tile_counter)
        _capi.check(_capi.load().vdi_render_launch(a, dv.stream_handle()))
        s = sums.cpu().numpy()
        return int(s[0]), int(s[1]), int(s[2])

    def render_per_pixel(self):
        """This rank's render again, with per-pixel counters (untimed):
        host (image, lists_visited, segs_intersected, lists_searched)."""
        t = self.t
        pp = [t.empty((self.out_rows, self.ow), dtype=t.int32, device="cuda") for _ in range(3)]
        a = render_args(self.dvdi, self.params.n_sg, self.w, self.h, self.gcam, self.aabb,
                        self.bufs.grid, self.grid_dims, self.gcam.near, self.gcam.far,
                        self.rcam, self.opts, self.image, per_pixel=pp, band=self.band)
        launch_zmask(a, self.zmask)
        set_tile_counter(a, self.tile_counter)
        _capi.check(_capi.load().vdi_render_launch(a, dv.stream_handle()))
        return (dv.to_host(self.image),) + tuple(dv.to_host(x) for x in pp)

    def generate_only(self, vol_dev=None, gather: bool = True):
        """This rank's volume prep + generation + partial grid (no exchange,
        no render), on the current stream."""
        vol_dev = self.vol_dev if vol_dev is None else vol_dev
        self.prep(vol_dev, gather)
        launch_generate(vol_dev, self.vt, self.vol.dims, self.lut_dev, self.gcam,
                        self.aabb, self.params, self.resolved, self.bufs, self.grid_dims,
                        band=self.gen_band, bricks=self.bricks, ess_max=self.ess_max,
                        cells=self.cells, sub=self.sub, rows=self.gen_range)

    def samples_executed(self) -> int:
        return int(self.bufs.samples.to(self.t.int64).sum().item())

    def render_stats(self):
        s = self.sums.cpu().numpy()
        return int(s[0]), int(s[1]), int(s[2])

    def host_vdi(self):
        """(counts, segs AoS, grid) on the host, natural row order (N=1)."""
        vdi = Vdi(self.w, self.h, self.params.n_sg, None, None, self.gcam, self.aabb,
                  _device=self.dvdi)
        return vdi.counts, vdi.segs, dv.to_host(self.bufs.grid).view(np.uint32)

    def e2e_stream(self, steps: int, warmup: int = 2, packed: bool = False):
        """End to end through the public FrameStream API: every frame uploads
        its volume from pinned host memory and reads its results (counts, AoS
        segs, AccelGrid, image) back to pinned host memory, overlapped with
        the neighbouring frames' kernels (stream.py). Time per frame over
        `steps` frames after `warmup` frames, max over ranks."""
        from .stream import FrameStream
        if self.bricked:
            raise NotImplementedError("e2e_stream: a bricked pipeline keeps only its voxel box "
                                      "resident; stream the box, not the full volume")
        t = self.t
        host = dv.pinned_numpy(self.vol.data.shape, self.vol.data.dtype)
        host[...] = self.vol.data
        fs = FrameStream(self, packed=packed)
        fs.run([host] * warmup)
        t.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
        d2h = []
        t0 = time.perf_counter()
        fs.run([host] * steps, on_result=lambda r: d2h.append(r.nbytes))
        t.cuda.synchronize()
        dt = (time.perf_counter() - t0) / steps
        if self.world > 1:
            x = t.tensor([dt], dtype=t.float64, device="cuda")
            self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX)
            dt = float(x.item())
        del fs
        mode = "FrameStream: H2D(i+1) | kernels(i) | D2H(i-1) overlapped"
        if packed:
            mode += "; VDI read back as its VDI1 bytes (encode_vdi, vdi.py:141)"
        return {"value": 2 * self.w * self.h / dt / 1e6, "unit": "Mrays/s",
                "h2d_bytes_per_step": int(fs_h2d(host, self.tf)),
                "d2h_bytes_per_step": int(np.mean(d2h)) if d2h else int(self._d2h_bytes()),
                "ms_per_step": dt * 1e3, "steps": steps, "mode": mode}

    def _d2h_bytes(self) -> int:
        n_sg = self.params.n_sg
        return (self.gen_rows * self.w * (4 + 24 * n_sg) + self.bufs.grid.numel() * 4
                + self.image.numel() * 8)

    def e2e(self, steps: int):
        """End to end through host buffers, one frame at a time: pinned volume
        H2D every step, the public generate_vdi / render_vdi (N=1) or the
        sharded pipeline (N>1), and the step's results read back to pinned
        host memory."""
        if self.bricked:
            raise NotImplementedError("e2e: a bricked pipeline keeps only its voxel box "
                                      "resident; upload the box, not the full volume")
        t = self.t
        vol = self.vol
        host = dv.pinned_numpy(vol.data.shape, vol.data.dtype)
        host[...] = vol.data
        from .volume import Volume
        pvol = Volume(dims=vol.dims, voxel_type=vol.voxel_type, spacing=vol.spacing,
                      data=host, value_range=vol.value_range)
        times, h2d, d2h = [], 0, 0
        # one untimed warm-up step, so the device workspace and the pinned host
        # result buffers come from the allocators' caches as in steady use
        for it in range(steps + 1):
            c = s = g = img = vdi = grid = None  # release the previous step's results
            t.cuda.synchronize()
            t0 = time.perf_counter()
            if self.world == 1:
                from .generate import generate_vdi
                from .raycast import render_vdi
                vdi, grid = generate_vdi(pvol, self.tf, self.gcam, self.params,
                                         cache_volume=False)
                c, s, g = vdi.counts, vdi.segs, grid.counts
                img = render_vdi(vdi, grid, self.rcam, self.opts)
                d2h = c.nbytes + s.nbytes + g.nbytes + img.data.nbytes
            else:
                self.vol_dev = dv.to_device(host)
                self.step()
                n_sg = self.params.n_sg
                aos = t.empty((self.gen_rows * self.w, n_sg * 6), dtype=t.float32,
                              device="cuda")
                _capi.check(_capi.load().vdi_segs_to_aos(
                    dv.ptr(self.bufs.segs), dv.ptr(aos), self.gen_rows * self.w, n_sg,
                    dv.stream_handle()))
                c = dv.to_host(self.bufs.counts, sync=False)
                s = dv.to_host(aos, sync=False)
                img = dv.to_host(self.image, sync=True)
                d2h = c.nbytes + s.nbytes + img.nbytes
            t.cuda.synchronize()
            if it > 0:
                times.append(time.perf_counter() - t0)
            h2d = host.nbytes + self.tf.lut.nbytes
        dt = float(np.mean(times))
        if self.world > 1:
            x = t.tensor([dt], dtype=t.float64, device="cuda")
            self.dist.all_reduce(x, op=self.dist.ReduceOp.MAX)
            dt = float(x.item())
        self.vol_dev, _ = dv.upload_volume(self.vol)
        return {"value": 2 * self.w * self.h / dt / 1e6, "unit": "Mrays/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": dt * 1e3, "steps": steps}


def fs_h2d(host, tf) -> int:
    """Input bytes a frame uploads: the volume (the LUT is uploaded once)."""
    return host.nbytes


def unshard_image(g_image, out_h: int, world: int):
    """Gathered band-interleaved image rows -> natural order (host numpy)."""
    idx = storage_rows(out_h, world)
    return np.asarray(g_image)[idx]
