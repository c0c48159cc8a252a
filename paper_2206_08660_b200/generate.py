"""VDI generation: drop-in for `vdikit.generate_vdi` (generate.py:444-479).

Same signature and return types; the per-ray bisection (Alg. 1 as the
reference implements it, generate.py:219-273), the front-to-back passes
(89-216) and the AccelGrid build (322-346) run as sm_100a kernels through
`vdi_gen_launch` / `vdi_grid_launch` (include/vdi_b200.h).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _capi
from . import device as dv
from .vdi import AccelGrid, DeviceVdi, Vdi, default_grid_dims

SQRT3 = 1.7320508075688772


def list_stride(n_sg: int) -> int:
    """Floats per list in the device list-SoA layout (vdi_list_stride)."""
    return (6 * n_sg + 3) & ~3


@dataclass(frozen=True)
class GenParams:
    """generate.py:28-50."""
    n_sg: int = 12
    delta: int | None = None
    epsilon: float = 1e-6
    gamma_init: float = 1e-5
    step: float | None = None
    ref_step: float | None = None
    alpha_early: float = 0.999

    def resolve(self, vol) -> tuple:
        step = self.step if self.step is not None else 0.5 * min(vol.spacing)
        lref = self.ref_step if self.ref_step is not None else step
        delta = max(1, int(0.15 * self.n_sg)) if self.delta is None else self.delta
        delta = min(delta, self.n_sg - 1)
        if not (0 < self.epsilon < 1):
            raise ValueError("epsilon must be in (0, 1)")
        if self.n_sg < 1:
            raise ValueError("n_sg must be >= 1")
        return delta, step, lref


@dataclass(frozen=True)
class GenStats:
    """generate.py:428-441, plus the executed-sample count per ray."""
    gammas: np.ndarray
    passes: np.ndarray
    wall_time_s: float
    samples: np.ndarray | None = None

    @property
    def max_passes(self) -> int:
        return int(self.passes.max())

    @property
    def mean_passes(self) -> float:
        active = self.passes[self.passes > 0]
        return float(active.mean()) if active.size else 0.0


def depth_consts(near: float, far: float) -> tuple:
    """generate.py:349-354."""
    return (far + near) / (far - near), 2.0 * far * near / (far - near)


def _mat(m) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(m, dtype=np.float64).reshape(16))


@dataclass
class GenBuffers:
    counts: object
    segs: object
    gammas: object
    passes: object
    samples: object
    workspace: object
    grid: object


def alloc_gen(width, rows, n_sg, grid_dims, stats=True):
    t = dv.torch()
    gx, gy, gz = grid_dims
    return GenBuffers(
        counts=t.empty((rows, width), dtype=t.int32, device="cuda"),
        segs=t.empty((rows * width, list_stride(n_sg)), dtype=t.float32, device="cuda"),
        gammas=t.empty((rows, width), dtype=t.float64, device="cuda") if stats else None,
        passes=t.empty((rows, width), dtype=t.int32, device="cuda") if stats else None,
        samples=t.empty((rows, width), dtype=t.int32, device="cuda") if stats else None,
        workspace=None,  # sized by vdi_gen_workspace_bytes at launch
        grid=t.empty((gz, gy, gx), dtype=t.int32, device="cuda"))


def gen_args(vol_dev, voxel_type, dims, lut_dev, cam, aabb, params_resolved, n_sg, eps,
             gamma_init, bufs: GenBuffers, band=(16, 1, 0), bricks=None,
             ess_max=-1.0, cells=None, sub=None, rows=None) -> _capi.VdiGenArgs:
    """sub: (origin, box dims, oob flag tensor) when vol_dev holds only a
    resident box of the dims volume (VdiGenArgs.sub_*). rows: (row_base,
    row_count), a contiguous range of image rows instead of the band map."""
    delta, step, lref = params_resolved
    width, height = cam.viewport
    a = _capi.VdiGenArgs()
    a.volume = dv.ptr(cells if cells is not None else vol_dev)
    a.lut = dv.ptr(lut_dev)
    a.brick_max = dv.ptr(bricks)
    a.ess_max = float(ess_max) if bricks is not None else -1.0
    a.brick_log2 = dv.BRICK_LOG2
    a.counts, a.segs = dv.ptr(bufs.counts), dv.ptr(bufs.segs)
    a.gammas, a.passes, a.samples = dv.ptr(bufs.gammas), dv.ptr(bufs.passes), dv.ptr(bufs.samples)
    _capi.fill(a.pv, _mat(cam.proj_view()))
    _capi.fill(a.inv_pv, _mat(cam.inv_proj_view()))
    _capi.fill(a.eye, np.asarray(cam.position, dtype=np.float64))
    _capi.fill(a.aabb, np.asarray(aabb, dtype=np.float64).reshape(6))
    a.eps, a.gamma_init, a.step, a.lref = float(eps), float(gamma_init), float(step), float(lref)
    a.voxel_type = _capi.VOXEL[voxel_type] | (_capi.VOXEL_CELLS if cells is not None else 0)
    a.nx, a.ny, a.nz = (int(v) for v in dims)
    a.lut_n = int(lut_dev.shape[0])
    a.width, a.height = int(width), int(height)
    a.n_sg, a.delta = int(n_sg), int(delta)
    a.band_rows, a.band_stride, a.band_offset = (int(v) for v in band)
    if sub is not None:
        org, box, oob = sub
        for k in range(3):
            a.sub_origin[k] = int(org[k])
            a.sub_dims[k] = int(box[k])
        a.sub_oob = dv.ptr(oob)
    if rows is not None:
        a.row_base, a.row_count = int(rows[0]), int(rows[1])
    return a


def grid_args(bufs: GenBuffers, cam, width, height, n_sg, grid_dims, band=(16, 1, 0),
              clear=True, rows=None) -> _capi.VdiGridArgs:
    pa, pb = depth_consts(cam.near, cam.far)
    g = _capi.VdiGridArgs()
    g.segs, g.counts, g.grid = dv.ptr(bufs.segs), dv.ptr(bufs.counts), dv.ptr(bufs.grid)
    g.near, g.far, g.proj_a, g.proj_b = float(cam.near), float(cam.far), pa, pb
    g.width, g.height, g.n_sg = int(width), int(height), int(n_sg)
    g.gx, g.gy, g.gz = (int(v) for v in grid_dims)
    g.band_rows, g.band_stride, g.band_offset = (int(v) for v in band)
    g.clear = int(clear)
    if rows is not None:
        g.row_base, g.row_count = int(rows[0]), int(rows[1])
    return g


def launch_generate(vol_dev, voxel_type, dims, lut_dev, cam, aabb, params, resolved,
                    bufs: GenBuffers, grid_dims, band=(16, 1, 0), stream=None,
                    split_events=None, workspace_bytes=None, bricks=None, ess_max=-1.0,
                    cells=None, sub=None, rows=None):
    """Enqueue generation + grid on the current stream (no sync, no alloc).
    split_events: optional CUDA events; [1] and [2] bracket the generation
    kernel (timing only). workspace_bytes overrides the recommended scratch
    size ("min" = the smallest accepted, which forces deferral rounds).
    cells: vdi_volume_cells() records of vol_dev to sample from (or None)."""
    L = _capi.load()
    s = dv.stream_handle() if stream is None else stream
    a = gen_args(vol_dev, voxel_type, dims, lut_dev, cam, aabb, resolved, params.n_sg,
                 params.epsilon, params.gamma_init, bufs, band, bricks, ess_max, cells, sub, rows)
    if workspace_bytes == "min":
        need = int(L.vdi_gen_workspace_min_bytes(a))
    elif workspace_bytes is not None:
        need = int(workspace_bytes)
    elif bufs.workspace is not None:
        # sized once (the recommendation depends on the free device memory)
        need = int(L.vdi_gen_workspace_min_bytes(a))
    else:
        need = int(L.vdi_gen_workspace_bytes(a))
    if bufs.workspace is None or bufs.workspace.numel() < need:
        bufs.workspace = dv.torch().empty(need, dtype=dv.torch().uint8, device="cuda")
    a.workspace, a.workspace_bytes = dv.ptr(bufs.workspace), int(bufs.workspace.numel())
    if split_events:
        split_events[1].record()
    _capi.check(L.vdi_gen_launch(a, s))
    if split_events:
        split_events[2].record()
    w, h = cam.viewport
    g = grid_args(bufs, cam, w, h, params.n_sg, grid_dims, band, rows=rows)
    _capi.check(L.vdi_grid_launch(g, s))


_shared_ws = {}


def shared_workspace(nbytes: int, min_bytes: int | None = None):
    """One generation scratch buffer per device, reused by every
    generate_vdi call (in stream order) and grown when a call needs more:
    the recommended size can be tens of GB, and allocating it per call
    thrashes the caching allocator. If `nbytes` cannot be allocated (other
    allocations on the device), falls back to `min_bytes`: the kernels then
    defer the rays that do not fit to later rounds (same results)."""
    t = dv.torch()
    dev = t.cuda.current_device()
    ws = _shared_ws.get(dev)
    if ws is None or ws.numel() < nbytes:
        _shared_ws.pop(dev, None)
        ws = None
        try:
            ws = t.empty(nbytes, dtype=t.uint8, device="cuda")
        except t.OutOfMemoryError:
            if min_bytes is None or min_bytes >= nbytes:
                raise
            t.cuda.empty_cache()
            ws = t.empty(min_bytes, dtype=t.uint8, device="cuda")
        _shared_ws[dev] = ws
    return ws


def release_workspace() -> None:
    """Drop the shared generation scratch (returns it to torch's cache)."""
    _shared_ws.clear()


def generate_vdi(vol, tf, cam, params: GenParams | None = None, grid_dims=None,
                 with_stats: bool = False, *, cache_volume: bool = True):
    """Generate a Vdi + AccelGrid from camera `cam` (one ray per viewport pixel).

    Mirrors generate.py:444-479. The returned Vdi / AccelGrid are device
    resident and materialise their numpy arrays on first access."""
    params = params or GenParams()
    resolved = params.resolve(vol)
    t = dv.require_cuda()
    width, height = cam.viewport
    if grid_dims is None:
        grid_dims = default_grid_dims(width, height)
    aabb = np.asarray(vol.aabb, dtype=np.float64)
    t_start = time.perf_counter()
    vol_dev, vt = dv.upload_volume(vol, cache=cache_volume)
    lut_dev = dv.upload_lut(tf.lut)
    bufs = alloc_gen(width, height, params.n_sg, grid_dims, stats=with_stats)
    a = gen_args(vol_dev, vt, vol.dims, lut_dev, cam, aabb, resolved, params.n_sg,
                 params.epsilon, params.gamma_init, bufs)
    L = _capi.load()
    bufs.workspace = shared_workspace(int(L.vdi_gen_workspace_bytes(a)),
                                      int(L.vdi_gen_workspace_min_bytes(a)))
    bricks = dv.volume_bricks(vol_dev, vt, vol.dims)
    cells = dv.volume_cells(vol_dev, vt, vol.dims) if dv.use_cells(vt, vol.dims) else None
    launch_generate(vol_dev, vt, vol.dims, lut_dev, cam, aabb, params, resolved, bufs,
                    grid_dims, bricks=bricks, ess_max=dv.ess_threshold(tf.lut), cells=cells)
    dev = DeviceVdi(counts=bufs.counts, segs=bufs.segs, sorted=True)
    vdi = Vdi(width=width, height=height, n_sg=params.n_sg, counts=None, segs=None,
              gen_camera=cam, volume_aabb=aabb, _device=dev)
    grid = AccelGrid(dims=grid_dims, counts=None, near=cam.near, far=cam.far,
                     _device=bufs.grid)
    if not with_stats:
        return vdi, grid
    t.cuda.current_stream().synchronize()
    wall = time.perf_counter() - t_start
    stats = GenStats(gammas=dv.to_host(bufs.gammas), passes=dv.to_host(bufs.passes),
                     wall_time_s=wall, samples=dv.to_host(bufs.samples))
    return vdi, grid, stats


# ------------------------------------------------------------ single rays (G14)

def terminate_check(seg_color, seg_alpha, sample_rgba, step_len, gamma) -> bool:
    """generate.py:357-368: True iff a new supersegment must start (a scalar
    predicate on host values, evaluated with the reference's expressions)."""
    import math
    a_adj = 1.0 - (1.0 - float(sample_rgba[3])) ** float(step_len)
    d = math.sqrt(sum((float(seg_color[c]) - float(sample_rgba[c]) * a_adj) ** 2
                      for c in range(3)))
    return d >= gamma


def _rays_array(rays) -> np.ndarray:
    out = np.empty((len(rays), 6), np.float64)
    for i, r in enumerate(rays):
        out[i, :3] = np.asarray(r.origin, np.float64)
        out[i, 3:] = np.asarray(r.dir, np.float64)
    return out


def gen_rays(rays, vol, tf, params: GenParams, cam, mode: int, gammas=None):
    """Batch of single-ray generations on the device (vdi_gen_rays): mode 0
    = find_gamma's bisection, 1 / 2 = one counting / capped pass at gammas.
    Returns host (counts, segs (n, n_sg, 6), gammas, passes, samples)."""
    t = dv.require_cuda()
    L = _capi.load()
    resolved = params.resolve(vol)
    n = len(rays)
    arr = _rays_array(rays)
    vol_dev, vt = dv.upload_volume(vol)
    lut_dev = dv.upload_lut(tf.lut)
    n_sg = params.n_sg
    bufs = GenBuffers(counts=t.zeros(max(n, 1), dtype=t.int32, device="cuda"),
                      segs=t.zeros((max(n, 1), list_stride(n_sg)), dtype=t.float32,
                                   device="cuda"),
                      gammas=t.zeros(max(n, 1), dtype=t.float64, device="cuda"),
                      passes=t.zeros(max(n, 1), dtype=t.int32, device="cuda"),
                      samples=t.zeros(max(n, 1), dtype=t.int32, device="cuda"),
                      workspace=None, grid=None)
    a = gen_args(vol_dev, vt, vol.dims, lut_dev, cam, np.asarray(vol.aabb, np.float64),
                 resolved, n_sg, params.epsilon, params.gamma_init, bufs)
    rays_dev = dv.to_device(arr)
    g_dev = dv.to_device(np.asarray(gammas, np.float64)) if gammas is not None else None
    _capi.check(L.vdi_gen_rays(a, dv.ptr(rays_dev), dv.ptr(g_dev), n, int(mode),
                               dv.stream_handle()))
    aos = t.empty((max(n, 1), n_sg * 6), dtype=t.float32, device="cuda")
    _capi.check(L.vdi_segs_to_aos(dv.ptr(bufs.segs), dv.ptr(aos), max(n, 1), n_sg,
                                  dv.stream_handle()))
    return (dv.to_host(bufs.counts)[:n], dv.to_host(aos).reshape(-1, n_sg, 6)[:n],
            dv.to_host(bufs.gammas)[:n], dv.to_host(bufs.passes)[:n],
            dv.to_host(bufs.samples)[:n])


def generate_list(ray, vol, tf, gamma: float, params: GenParams, cam, capped: bool = False):
    """generate.py:371-387: one generation pass along `ray` at `gamma`;
    returns (count, segments (n_sg, 6) f32, exceeded)."""
    c, s, _, _, _ = gen_rays([ray], vol, tf, params, cam, 2 if capped else 1, [float(gamma)])
    n = int(c[0])
    return min(n, params.n_sg), s[0], n > params.n_sg


def find_gamma(ray, vol, tf, params: GenParams, cam):
    """generate.py:390-407: the per-ray bisection; returns (gamma, count,
    segments, passes) (segments past `count` are zero)."""
    c, s, g, p, _ = gen_rays([ray], vol, tf, params, cam, 0)
    return float(g[0]), int(c[0]), s[0], int(p[0])
