"""Kernel-side band maps of the multi-GPU path, on one GPU.

Two "ranks" are emulated sequentially (no kernel waits on another): each
generates its interleaved 16-row bands into a padded shard, the shards are
concatenated exactly as an NCCL all-gather would lay them out, and the render
kernel reads that band-interleaved VDI through its storage-row map while
writing only its own output bands. Everything must equal the unsharded path
bit for bit.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2206_08660_b200 import _capi, shard, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200.generate import GenParams, alloc_gen, launch_generate  # noqa: E402
from paper_2206_08660_b200.raycast import RenderOptions, render_args  # noqa: E402
from paper_2206_08660_b200.vdi import DeviceVdi, default_grid_dims  # noqa: E402


@pytest.mark.parametrize("world", [2, 3])
def test_banded_generate_and_render_match_unsharded(world):
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    # a non-multiple-of-16 height exercises ragged bands
    from paper_2206_08660_b200.camera import Camera
    gcam = Camera(gcam.position, gcam.orientation, gcam.fov_y, gcam.near, gcam.far, (128, 100))
    rcam = Camera(rcam.position, rcam.orientation, rcam.fov_y, rcam.near, rcam.far, (120, 90))
    params = GenParams(n_sg=n_sg)
    res = params.resolve(vol)
    w, h = gcam.viewport
    dims = default_grid_dims(w, h)
    vd, vt = dv.upload_volume(vol)
    lut = dv.upload_lut(tf.lut)
    bricks = dv.volume_bricks(vd, vt, vol.dims)
    ess = dv.ess_threshold(tf.lut)

    full = alloc_gen(w, h, n_sg, dims)
    launch_generate(vd, vt, vol.dims, lut, gcam, vol.aabb, params, res, full, dims,
                    bricks=bricks, ess_max=ess)

    per = shard.rows_per_rank(h, world)
    shards, grid = [], torch.zeros_like(full.grid)
    for r in range(world):
        b = alloc_gen(w, per, n_sg, dims)
        b.counts.zero_()
        b.segs.zero_()
        launch_generate(vd, vt, vol.dims, lut, gcam, vol.aabb, params, res, b, dims,
                        band=(16, world, r), bricks=bricks, ess_max=ess)
        grid += b.grid  # the NCCL all-reduce
        shards.append(b)
    g_counts = torch.cat([b.counts for b in shards])      # the NCCL all-gathers
    g_segs = torch.cat([b.segs for b in shards])
    st = torch.from_numpy(shard.storage_rows(h, world)).cuda()
    assert torch.equal(g_counts[st], full.counts)
    assert torch.equal(g_segs.view(-1, w, g_segs.shape[1])[st].reshape(h * w, -1), full.segs)
    assert torch.equal(grid, full.grid)

    # render: natural layout vs band-interleaved VDI + banded output rows
    opts = RenderOptions()
    ow, oh = rcam.viewport
    L = _capi.load()
    ref_img = torch.zeros((oh, ow, 4), dtype=torch.float64, device="cuda")
    a = render_args(DeviceVdi(full.counts, full.segs), n_sg, w, h, gcam, vol.aabb, full.grid,
                    dims, gcam.near, gcam.far, rcam, opts, ref_img)
    _capi.check(L.vdi_render_launch(a, dv.stream_handle()))
    dvdi = DeviceVdi(g_counts, g_segs, 16, world, per)
    oper = shard.rows_per_rank(oh, world)
    parts = []
    for r in range(world):
        img = torch.zeros((oper, ow, 4), dtype=torch.float64, device="cuda")
        a = render_args(dvdi, n_sg, w, h, gcam, vol.aabb, grid, dims, gcam.near, gcam.far,
                        rcam, opts, img, band=(16, world, r))
        _capi.check(L.vdi_render_launch(a, dv.stream_handle()))
        parts.append(img)
    g_img = torch.cat(parts)[torch.from_numpy(shard.storage_rows(oh, world)).cuda()]
    assert torch.equal(g_img, ref_img)
