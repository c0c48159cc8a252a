"""Empty-list skipping in the render DDA: the
8x8-list tile bitmap (vdi_list_tiles) lets the render step through lists of
empty tiles without reading their counts. The image and every per-pixel
counter (lists visited / searched, supersegments intersected) must equal
the render without the bitmap bit for bit, and the bitmap must equal the
tile occupancy of the counts.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import _capi, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200.raycast import (alloc_list_tiles, launch_list_tiles,  # noqa: E402
                                           render_args)


def _tiles_ref(counts):
    h, w = counts.shape
    ty, tx = -(-h // 8), -(-w // 8)
    wpr = -(-tx // 32)
    occ = np.zeros((ty, wpr * 32), bool)
    for y in range(ty):
        for x in range(tx):
            occ[y, x] = (counts[8 * y:8 * y + 8, 8 * x:8 * x + 8] > 0).any()
    bits = occ.reshape(ty, wpr, 32).astype(np.uint64) << np.arange(32, dtype=np.uint64)
    return bits.sum(axis=2).astype(np.uint32).reshape(-1)


@pytest.mark.parametrize("cfg,angle", [("C2", 15.0), ("C2", 40.0), ("C3", 15.0)])
def test_tiles_exact(cfg, angle):
    vol, tf, gcam, rcam, n_sg = synth.config(cfg)
    rcam = synth.sweep_camera(vol, angle, gcam.viewport, synth.CONFIGS[cfg][4])
    vdi, grid = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg))
    d = vdi.device()
    ow, oh = rcam.viewport
    L = _capi.load()
    outs = []
    for use in (False, True):
        image = torch.empty((oh, ow, 4), dtype=torch.float64, device="cuda")
        pp = [torch.empty((oh, ow), dtype=torch.int32, device="cuda") for _ in range(3)]
        a = render_args(d, n_sg, vdi.width, vdi.height, gcam, vdi.volume_aabb, grid.device(),
                        grid.dims, grid.near, grid.far, rcam, vb.RenderOptions(), image,
                        per_pixel=pp)
        if use:
            tiles = alloc_list_tiles(vdi.width, vdi.height)
            launch_list_tiles(a, tiles)
            got = tiles.cpu().numpy().view(np.uint32)
            np.testing.assert_array_equal(got, _tiles_ref(d.counts.cpu().numpy()))
        _capi.check(L.vdi_render_launch(a, dv.stream_handle()))
        torch.cuda.synchronize()
        outs.append([image.cpu().numpy()] + [x.cpu().numpy() for x in pp])
    for x, y in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(x, y)
    assert outs[0][1].sum() > 0


def _zmask_ref(grid):
    gz, gy, gx = grid.shape
    bits = (grid > 0).astype(np.uint64) << np.arange(gz, dtype=np.uint64)[:, None, None]
    return bits.sum(axis=0).astype(np.uint64).reshape(-1)


@pytest.mark.parametrize("cfg,angle", [("C2", 15.0), ("C2", 40.0), ("C3", 15.0)])
def test_zmask_exact(cfg, angle):
    """The ESS test through the grid's per-column slab words
    (VdiRenderArgs.grid_zmask) gives the image and every counter of the
    cell-by-cell test (raycast.py:359-370)."""
    from paper_2206_08660_b200.raycast import alloc_zmask, launch_zmask
    vol, tf, gcam, rcam, n_sg = synth.config(cfg)
    rcam = synth.sweep_camera(vol, angle, gcam.viewport, synth.CONFIGS[cfg][4])
    vdi, grid = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg))
    d = vdi.device()
    ow, oh = rcam.viewport
    L = _capi.load()
    outs = []
    for use in (False, True):
        image = torch.empty((oh, ow, 4), dtype=torch.float64, device="cuda")
        pp = [torch.empty((oh, ow), dtype=torch.int32, device="cuda") for _ in range(3)]
        a = render_args(d, n_sg, vdi.width, vdi.height, gcam, vdi.volume_aabb, grid.device(),
                        grid.dims, grid.near, grid.far, rcam, vb.RenderOptions(), image,
                        per_pixel=pp)
        if use:
            zm = alloc_zmask(grid.dims)
            launch_zmask(a, zm)
            got = zm.cpu().numpy().view(np.uint64)
            np.testing.assert_array_equal(got, _zmask_ref(grid.device().cpu().numpy()))
        _capi.check(L.vdi_render_launch(a, dv.stream_handle()))
        torch.cuda.synchronize()
        outs.append([image.cpu().numpy()] + [x.cpu().numpy() for x in pp])
    for x, y in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(x, y)
    assert outs[0][3].sum() > 0


@pytest.mark.parametrize("cfg,angle", [("C2", 15.0), ("C2", 120.0), ("C2", 180.0),
                                       ("C3", 15.0), ("C3", 100.0)])
def test_search_first_shading_exact(cfg, angle):
    """Search-first shading (VdiRenderArgs.lists_sorted, generated VDIs,
    counters not exact) against the reference's ESS-then-search order: the
    same image and the same lists_visited / supersegments_intersected per
    pixel, forward chords (15 deg) and views behind the volume (reverse
    chords take the reference order); with and without the per-list depth
    ranges (VdiRenderArgs.list_range) that skip lists the chord misses."""
    from paper_2206_08660_b200.raycast import (alloc_ranges, alloc_zmask, launch_ranges,
                                               launch_zmask)
    vol, tf, gcam, rcam, n_sg = synth.config(cfg)
    rcam = synth.sweep_camera(vol, angle, gcam.viewport, synth.CONFIGS[cfg][4])
    vdi, grid = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg))
    d = vdi.device()
    assert d.sorted
    ow, oh = rcam.viewport
    L = _capi.load()
    outs = []
    for exact, ranged in ((True, False), (False, False), (False, True)):
        image = torch.empty((oh, ow, 4), dtype=torch.float64, device="cuda")
        pp = [torch.zeros((oh, ow), dtype=torch.int32, device="cuda") for _ in range(3)]
        a = render_args(d, n_sg, vdi.width, vdi.height, gcam, vdi.volume_aabb, grid.device(),
                        grid.dims, grid.near, grid.far, rcam, vb.RenderOptions(), image,
                        per_pixel=pp, counters_exact=exact)
        assert a.lists_sorted == 1
        zm = alloc_zmask(grid.dims)
        launch_zmask(a, zm)
        if ranged:
            rg = alloc_ranges(d.counts.numel())
            launch_ranges(a, rg, d.counts.numel())
        _capi.check(L.vdi_render_launch(a, dv.stream_handle()))
        torch.cuda.synchronize()
        outs.append([image.cpu().numpy()] + [x.cpu().numpy() for x in pp[:2]])
    for other in outs[1:]:
        for x, y in zip(outs[0], other):
            np.testing.assert_array_equal(x, y)
    assert outs[0][1].sum() > 0
    # the public API without stats takes the search-first path
    img = vb.render_vdi(vdi, grid, rcam)
    np.testing.assert_array_equal(img.data, outs[0][0])


def _ranges_ref(counts, segs_soa, n_sg):
    n = counts.size
    fr = segs_soa[:, 4 * n_sg:5 * n_sg]
    bk = segs_soa[:, 5 * n_sg:6 * n_sg]
    out = np.empty((n, 2), np.float32)
    for i, c in enumerate(counts.reshape(-1)):
        f, b = fr[i, :c], bk[i, :c]
        if np.isnan(f).any() or np.isnan(b).any():
            out[i] = (-np.inf, np.inf)
        elif c == 0:
            out[i] = (np.inf, -np.inf)
        else:
            out[i] = (f.min(), b.max())
    return out


def test_list_ranges_kernel():
    """vdi_list_ranges: (min front, max back) per list, the empty and NaN
    sentinels, counts beyond n_sg clamped."""
    from paper_2206_08660_b200.raycast import alloc_ranges
    rng = np.random.default_rng(5)
    n_sg, n = 6, 5000
    stride = (6 * n_sg + 3) & ~3
    segs = rng.random((n, stride)).astype(np.float32)
    counts = rng.integers(0, n_sg + 1, n).astype(np.int32)
    segs[7, 4 * n_sg + 1] = np.nan
    counts[7] = 3
    segs[8, 5 * n_sg + 4] = np.nan
    counts[8] = 4  # NaN beyond the count: ignored
    want = _ranges_ref(counts, segs, n_sg)
    out = alloc_ranges(n)
    _capi.check(_capi.load().vdi_list_ranges(dv.ptr(dv.to_device(segs)),
                                             dv.ptr(dv.to_device(counts)), n, n_sg,
                                             dv.ptr(out), dv.stream_handle()))
    np.testing.assert_array_equal(out.cpu().numpy().reshape(n, 2), want)
    assert np.isinf(want[7]).all() and want[8, 0] < want[8, 1]


@pytest.mark.parametrize("cfg,angle", [("C2", 15.0), ("C2", 180.0), ("C3", 15.0)])
def test_dynamic_tiles_exact(cfg, angle):
    """The resident render grid taking tiles from a counter
    (VdiRenderArgs.tile_counter) gives the image, the per-pixel counters and
    the counter sums of the one-tile-per-warp grid, and leaves the counter
    zeroed for the next launch (three launches on one counter)."""
    from paper_2206_08660_b200.raycast import alloc_zmask, launch_zmask
    vol, tf, gcam, rcam, n_sg = synth.config(cfg)
    rcam = synth.sweep_camera(vol, angle, gcam.viewport, synth.CONFIGS[cfg][4])
    vdi, grid = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg))
    d = vdi.device()
    ow, oh = rcam.viewport
    L = _capi.load()
    counter = torch.zeros(2, dtype=torch.int32, device="cuda")
    outs = []
    for dyn in (False, True, True, True):
        image = torch.empty((oh, ow, 4), dtype=torch.float64, device="cuda")
        pp = [torch.zeros((oh, ow), dtype=torch.int32, device="cuda") for _ in range(3)]
        sums = torch.zeros(3, dtype=torch.int64, device="cuda")
        a = render_args(d, n_sg, vdi.width, vdi.height, gcam, vdi.volume_aabb, grid.device(),
                        grid.dims, grid.near, grid.far, rcam, vb.RenderOptions(), image,
                        per_pixel=pp, stat_sums=sums)
        zm = alloc_zmask(grid.dims)
        launch_zmask(a, zm)
        a.tile_counter = dv.ptr(counter) if dyn else None
        _capi.check(L.vdi_render_launch(a, dv.stream_handle()))
        torch.cuda.synchronize()
        assert counter.cpu().tolist() == [0, 0]
        outs.append([image.cpu().numpy()] + [x.cpu().numpy() for x in pp] + [sums.cpu().numpy()])
    for other in outs[1:]:
        for x, y in zip(outs[0], other):
            np.testing.assert_array_equal(x, y)
    assert outs[0][4][0] == outs[0][1].sum() > 0
