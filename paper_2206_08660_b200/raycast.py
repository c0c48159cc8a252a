"""Novel-view VDI rendering: drop-in for `vdikit.render_vdi` (raycast.py:459-491).

The per-pixel NDC DDA, ESS test, Alg. 2 seeded search and Eq. 2 compositing
(raycast.py:275-456) run in `vdi_render_launch` (include/vdi_b200.h).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _capi
from . import device as dv
from .generate import depth_consts, _mat
from .image import Image


@dataclass(frozen=True)
class RenderOptions:
    """raycast.py:28-36."""
    use_ess: bool = True
    early_term_alpha: float = 0.999
    background: tuple = (0.0, 0.0, 0.0, 1.0)

    def __post_init__(self):
        if not (0.0 < self.early_term_alpha <= 1.0):
            raise ValueError("early_term_alpha must be in (0, 1]")


@dataclass(frozen=True)
class RenderStats:
    """raycast.py:39-43 (+ lists searched, a counter the reference lacks)."""
    lists_visited: int
    supersegments_intersected: int
    frame_ms: float
    lists_searched: int = -1


def opacity_correct(alpha: float, l: float) -> float:
    """raycast.py:46-48."""
    return 1.0 - (1.0 - alpha) ** l


def render_args(dvdi, n_sg, vdi_w, vdi_h, gen_cam, aabb, grid_dev, grid_dims, grid_near,
                grid_far, cam_new, opts, image, per_pixel=None, stat_sums=None,
                band=(16, 1, 0), counters_exact=None) -> _capi.VdiRenderArgs:
    """counters_exact: count lists_searched exactly (the reference's ESS-then-
    search order); default: exactly when per-pixel counters or stat sums are
    requested. Image, lists_visited and segs_intersected are exact either
    way."""
    a = _capi.VdiRenderArgs()
    a.segs, a.counts, a.grid, a.image = (dv.ptr(dvdi.segs), dv.ptr(dvdi.counts),
                                         dv.ptr(grid_dev), dv.ptr(image))
    if per_pixel is not None:
        a.lists_visited, a.segs_intersected, a.lists_searched = (dv.ptr(x) for x in per_pixel)
    a.stat_sums = dv.ptr(stat_sums)
    _capi.fill(a.gen_pv, _mat(gen_cam.proj_view()))
    _capi.fill(a.gen_inv_pv, _mat(gen_cam.inv_proj_view()))
    _capi.fill(a.new_inv_pv, _mat(cam_new.inv_proj_view()))
    _capi.fill(a.eye, np.asarray(cam_new.position, dtype=np.float64))
    _capi.fill(a.aabb, np.asarray(aabb, dtype=np.float64).reshape(6))
    _capi.fill(a.bg, np.asarray(opts.background, dtype=np.float64))
    pa, pb = depth_consts(gen_cam.near, gen_cam.far)
    a.near, a.far, a.proj_a, a.proj_b = float(grid_near), float(grid_far), pa, pb
    a.early_term = float(opts.early_term_alpha)
    a.vdi_w, a.vdi_h, a.n_sg = int(vdi_w), int(vdi_h), int(n_sg)
    a.gx, a.gy, a.gz = (int(v) for v in grid_dims)
    a.out_w, a.out_h = (int(v) for v in cam_new.viewport)
    a.use_ess = int(bool(opts.use_ess))
    a.vdi_band_rows, a.vdi_band_world = int(dvdi.band_rows), int(dvdi.world)
    a.vdi_rows_per_rank = int(dvdi.rows_per_rank)
    a.band_rows, a.band_stride, a.band_offset = (int(v) for v in band)
    a.lists_sorted = int(bool(getattr(dvdi, "sorted", False)))
    a.vdi_row_map = dv.ptr(getattr(dvdi, "row_map", None))
    if counters_exact is None:
        counters_exact = per_pixel is not None or stat_sums is not None
    a.counters_exact = int(bool(counters_exact))
    return a


def use_list_tiles() -> bool:
    """Empty-tile skipping in the render DDA (VdiRenderArgs.list_tiles). Exact,
    but off by default: the counts it avoids reading are L2-resident (8 MB at
    1080p) and the staging costs more than it saves on C2-C5 (render C3 0.98
    -> 1.02 ms, C5 11.1 -> 11.8 ms). tuning.TUNING.list_tiles turns it on."""
    from .tuning import TUNING
    return bool(TUNING.list_tiles)


def alloc_list_tiles(vdi_w: int, vdi_h: int):
    words = int(_capi.load().vdi_list_tiles_words(int(vdi_w), int(vdi_h)))
    return dv.torch().empty(max(words, 1), dtype=dv.torch().int32, device="cuda")


def launch_list_tiles(a: _capi.VdiRenderArgs, tiles, stream=None) -> None:
    """Occupancy bitmap of 8x8-list tiles for the render (vdi_list_tiles),
    from the VDI counts `a` points at; sets a.list_tiles."""
    _capi.check(_capi.load().vdi_list_tiles(a, dv.ptr(tiles), dv.stream_handle()
                                            if stream is None else stream))
    a.list_tiles = dv.ptr(tiles)


def alloc_zmask(grid_dims):
    """Per-column slab words of an AccelGrid (vdi_grid_zmask), or None when
    gz > 64 (the render then reads the grid cells directly)."""
    gx, gy, gz = (int(v) for v in grid_dims)
    if gz > 64:
        return None
    return dv.torch().empty(gx * gy, dtype=dv.torch().int64, device="cuda")


def launch_zmask(a: _capi.VdiRenderArgs, zmask, stream=None) -> None:
    """Build the slab words of the grid `a` points at; sets a.grid_zmask."""
    if zmask is None:
        a.grid_zmask = None
        return
    _capi.check(_capi.load().vdi_grid_zmask(a.grid, a.gx, a.gy, a.gz, dv.ptr(zmask),
                                            dv.stream_handle() if stream is None else stream))
    a.grid_zmask = dv.ptr(zmask)


def use_list_ranges(a: _capi.VdiRenderArgs) -> bool:
    """Per-list depth ranges (VdiRenderArgs.list_range) pay only where the
    kernel reads them: sorted lists without exact search counters."""
    from .tuning import TUNING
    return bool(TUNING.list_ranges) and bool(a.lists_sorted) and not a.counters_exact


def alloc_ranges(n_lists: int):
    return dv.torch().empty(2 * max(int(n_lists), 1), dtype=dv.torch().float32, device="cuda")


def launch_ranges(a: _capi.VdiRenderArgs, ranges, n_lists: int, stream=None) -> None:
    """(min front, max back) of every storage list of the VDI `a` points at
    (vdi_list_ranges); sets a.list_range (None: a.list_range = NULL)."""
    if ranges is None:
        a.list_range = None
        return
    _capi.check(_capi.load().vdi_list_ranges(a.segs, a.counts, int(n_lists), a.n_sg,
                                             dv.ptr(ranges), dv.stream_handle()
                                             if stream is None else stream))
    a.list_range = dv.ptr(ranges)


def alloc_tile_counter():
    """The render's tile counter (VdiRenderArgs.tile_counter), or None when
    tuning.TUNING.dyn_tiles is off. Zeroed here; every launch leaves it zero."""
    from .tuning import TUNING
    if not TUNING.dyn_tiles:
        return None
    return dv.torch().zeros(2, dtype=dv.torch().int32, device="cuda")


def set_tile_counter(a: _capi.VdiRenderArgs, counter) -> None:
    a.tile_counter = dv.ptr(counter) if counter is not None else None


def launch_render(vdi, grid, cam_new, opts, image, per_pixel=None, stat_sums=None,
                  band=(16, 1, 0), stream=None):
    """Enqueue one render on the current stream (no sync; the grid's slab
    words and, if enabled, a tile bitmap are allocated per call)."""
    a = render_args(vdi.device(), vdi.n_sg, vdi.width, vdi.height, vdi.gen_camera,
                    vdi.volume_aabb, grid.device(), grid.dims, grid.near, grid.far, cam_new,
                    opts, image, per_pixel, stat_sums, band)
    s = dv.stream_handle() if stream is None else stream
    tiles = None
    if use_list_tiles():
        tiles = alloc_list_tiles(vdi.width, vdi.height)
        launch_list_tiles(a, tiles, s)
    zmask = alloc_zmask(grid.dims) if opts.use_ess else None
    launch_zmask(a, zmask, s)
    ranges = None
    if use_list_ranges(a):
        n_lists = vdi.device().counts.numel()
        ranges = alloc_ranges(n_lists)
        launch_ranges(a, ranges, n_lists, s)
    counter = alloc_tile_counter()
    set_tile_counter(a, counter)
    _capi.check(_capi.load().vdi_render_launch(a, s))
    # they must outlive the enqueued render
    image._keep_tiles = (tiles, zmask, ranges, counter)


def _as_device_vdi(vdi):
    """Accept our Vdi or any object with the reference Vdi's attributes (a
    frozen vdikit.Vdi of numpy arrays). A reference object is uploaded on
    every call -- no device copy is cached on it, so an array the caller
    mutates in place is never rendered stale."""
    if hasattr(vdi, "device"):
        return vdi
    from .vdi import Vdi
    return Vdi(vdi.width, vdi.height, vdi.n_sg, vdi.counts, vdi.segs, vdi.gen_camera,
               vdi.volume_aabb)


def _as_device_grid(grid):
    if hasattr(grid, "device"):
        return grid
    from .vdi import AccelGrid
    return AccelGrid(grid.dims, grid.counts, grid.near, grid.far)


def render_vdi(vdi, grid, cam_new, opts: RenderOptions | None = None,
               with_stats: bool = False):
    """Render a VDI from a novel viewpoint; returns Image (and RenderStats)."""
    opts = opts or RenderOptions()
    t = dv.require_cuda()
    vdi = _as_device_vdi(vdi)
    grid = _as_device_grid(grid)
    out_w, out_h = cam_new.viewport
    image = t.empty((out_h, out_w, 4), dtype=t.float64, device="cuda")
    sums = t.zeros(3, dtype=t.int64, device="cuda") if with_stats else None
    t_start = time.perf_counter()
    ev0 = ev1 = None
    if with_stats:
        ev0, ev1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        ev0.record()
    launch_render(vdi, grid, cam_new, opts, image, stat_sums=sums)
    if with_stats:
        ev1.record()
    img = Image.from_array(dv.to_host(image))
    if not with_stats:
        return img
    s = dv.to_host(sums)
    ms = ev0.elapsed_time(ev1) if ev0 is not None else (time.perf_counter() - t_start) * 1e3
    return img, RenderStats(lists_visited=int(s[0]), supersegments_intersected=int(s[1]),
                            frame_ms=float(ms), lists_searched=int(s[2]))


def find_first_supersegment(seg_list, d_entry: float, d_exit: float, p: int = -1):
    """raycast.py:144-156 on the device (batch of one query)."""
    res = find_first_batch(np.asarray(seg_list, np.float32).reshape(1, -1, 6),
                           [len(np.asarray(seg_list).reshape(-1, 6))], [d_entry], [d_exit], [p])
    idx, seed = int(res[0][0]), int(res[1][0])
    return (None if idx < 0 else idx), seed


def find_first_batch(lists, counts, d_entry, d_exit, seeds):
    """Alg. 2 search for many independent queries: lists (n, n_max, 6) f32."""
    t = dv.require_cuda()
    lists = np.asarray(lists, np.float32)
    n, n_max = lists.shape[0], lists.shape[1]
    fr = dv.to_device(np.ascontiguousarray(lists[..., 0]))
    bk = dv.to_device(np.ascontiguousarray(lists[..., 1]))
    cnt = dv.to_device(np.asarray(counts, np.int32))
    de = dv.to_device(np.asarray(d_entry, np.float64))
    dx = dv.to_device(np.asarray(d_exit, np.float64))
    sd = dv.to_device(np.asarray(seeds, np.int32))
    oi = t.empty(n, dtype=t.int32, device="cuda")
    osd = t.empty(n, dtype=t.int32, device="cuda")
    _capi.check(_capi.load().vdi_find_first_batch(
        dv.ptr(fr), dv.ptr(bk), dv.ptr(cnt), int(n_max), dv.ptr(de), dv.ptr(dx), dv.ptr(sd),
        dv.ptr(oi), dv.ptr(osd), int(n), dv.stream_handle()))
    return dv.to_host(oi), dv.to_host(osd)


# ------------------------------------------------------- test-facing (R9, R10)

def composite_lists(vdi, opts: RenderOptions | None = None) -> Image:
    """raycast.py:494-518: the identity-view oracle -- each list's stored
    supersegments composited front to back, no traversal, no length
    correction -- on the device (vdi_composite_lists)."""
    opts = opts or RenderOptions()
    t = dv.require_cuda()
    vdi = _as_device_vdi(vdi)
    d = vdi.device()
    counts, segs = d.counts, d.segs
    if d.world > 1:
        from .vdi import unshard_rows
        counts, segs = unshard_rows(d, vdi.height, vdi.width)
    img = t.empty((vdi.height, vdi.width, 4), dtype=t.float64, device="cuda")
    bg = np.ascontiguousarray(np.asarray(opts.background, np.float64))
    _capi.check(_capi.load().vdi_composite_lists(
        dv.ptr(segs), dv.ptr(counts), vdi.width, vdi.height, vdi.n_sg,
        float(opts.early_term_alpha), bg.ctypes.data, dv.ptr(img), dv.stream_handle()))
    return Image.from_array(dv.to_host(img))


def dda_traverse(a0, a1, width: int, height: int):
    """raycast.py:225-234: the list cells an NDC chord visits, with the
    per-cell entry / exit NDC z (vdi_dda_cells)."""
    t = dv.require_cuda()
    cap = int(width) + int(height) + 4
    ch = dv.to_device(np.concatenate([np.asarray(a0, np.float64).reshape(3),
                                      np.asarray(a1, np.float64).reshape(3)]))
    cells = t.empty((cap, 2), dtype=t.int32, device="cuda")
    zs = t.empty((cap, 4), dtype=t.float64, device="cuda")
    n = t.empty(1, dtype=t.int32, device="cuda")
    _capi.check(_capi.load().vdi_dda_cells(dv.ptr(ch), 1, int(width), int(height), cap,
                                           dv.ptr(cells), dv.ptr(zs), dv.ptr(n),
                                           dv.stream_handle()))
    k = int(dv.to_host(n)[0])
    c, z = dv.to_host(cells), dv.to_host(zs)
    return [((int(c[i, 0]), int(c[i, 1])), float(z[i, 0]), float(z[i, 1])) for i in range(k)]


def project_ray_to_ndc(ray, gen_cam, volume_aabb):
    """raycast.py:237-255: the ray clipped to the volume box and the
    generation frustum, as an NDC chord (a0, a1), or None."""
    t = dv.require_cuda()
    r = dv.to_device(np.concatenate([np.asarray(ray.origin, np.float64).reshape(3),
                                     np.asarray(ray.dir, np.float64).reshape(3)]))
    out = t.empty(6, dtype=t.float64, device="cuda")
    hit = t.empty(1, dtype=t.int32, device="cuda")
    pv = np.ascontiguousarray(_mat(gen_cam.proj_view()))
    bb = np.ascontiguousarray(np.asarray(volume_aabb, np.float64).reshape(6))
    _capi.check(_capi.load().vdi_project_rays(dv.ptr(r), 1, pv.ctypes.data, bb.ctypes.data,
                                              dv.ptr(out), dv.ptr(hit), dv.stream_handle()))
    if not int(dv.to_host(hit)[0]):
        return None
    o = dv.to_host(out)
    return o[:3].copy(), o[3:].copy()
