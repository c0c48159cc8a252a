"""Volume bricked across GPUs (BASELINE C5 "bricked across
8 x B200"): each rank generates a contiguous band of rows with only the
voxel box its rays sample resident (shard.band_volume_box, VdiGenArgs.sub_*).

One GPU is available here, so the ranks' generations run one after another
(they are independent: no rank waits on another; the exchange after them is
covered by tests/test_multirank.py over gloo). Each rank's lists must equal,
bit for bit, the same rows of the full-volume generation, with no sample
outside the resident box (sub_oob == 0) and a box well below the volume.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import generate as gen  # noqa: E402
from paper_2206_08660_b200 import shard, synth  # noqa: E402


def _check(cfg, world, box_volume=None, max_frac=0.75, balanced=False):
    vol, tf, gcam, rcam, n_sg = synth.config(cfg)
    params = vb.GenParams(n_sg=n_sg)
    vdi, grid, st = vb.generate_vdi(vol, tf, gcam, params, with_stats=True)
    d = vdi.device()
    torch.cuda.synchronize()
    gen.release_workspace()  # the ranks below allocate their own (large) workspaces
    torch.cuda.empty_cache()
    w, h = gcam.viewport
    full_bytes = int(np.prod(vol.dims)) * (1 if vol.voxel_type == "u8" else 4)
    grid_sum = torch.zeros_like(grid.device())
    bounds = shard.balance_bands(st.samples.sum(axis=1), world) if balanced else None
    shards = []
    for r in range(world):
        p = shard.Pipeline(vol, tf, gcam, rcam, params, world=world, rank=r, bricked=True,
                           box_volume=box_volume, band_bounds=bounds)
        p.generate_only()
        torch.cuda.synchronize()
        assert int(p.oob.item()) == 0, f"rank {r}: sample outside the resident box {p.box}"
        res = p.vol_dev.numel() * p.vol_dev.element_size()
        assert res <= max_frac * full_bytes, (r, p.box)
        if balanced:
            r0, n = p.gen_range
            per = p.gen_rows
            shards.append((p.bufs.counts.clone(), p.bufs.segs.clone()))
        else:
            r0 = r * p.gen_band_rows
            n = min(h, r0 + p.gen_band_rows) - r0
        assert torch.equal(p.bufs.counts[:n], d.counts[r0:r0 + n]), r
        seg_rows = p.bufs.segs.view(-1, w, p.bufs.segs.shape[1])[:n]
        full_rows = d.segs.view(-1, w, d.segs.shape[1])[r0:r0 + n]
        assert torch.equal(seg_rows, full_rows), r
        assert torch.equal(p.bufs.samples[:n].cpu(), torch.from_numpy(st.samples[r0:r0 + n])), r
        grid_sum += p.bufs.grid
        del p
        torch.cuda.empty_cache()
    assert torch.equal(grid_sum, grid.device())  # the all-reduce of the partial grids
    if balanced:
        # the all-gathered storage (shards padded to the tallest band), read by
        # the render through VdiRenderArgs.vdi_row_map: the natural render
        from paper_2206_08660_b200 import device as dv
        from paper_2206_08660_b200.vdi import DeviceVdi
        g_counts = torch.cat([c for c, _ in shards])
        g_segs = torch.cat([s_ for _, s_ in shards])
        rmap = dv.to_device(shard.row_storage_map(bounds, per))
        gvdi = vb.Vdi(w, h, n_sg, None, None, gcam, vol.aabb,
                      _device=DeviceVdi(g_counts, g_segs, sorted=True, row_map=rmap))
        ref_img = vb.render_vdi(vdi, grid, rcam).data
        assert np.array_equal(vb.render_vdi(gvdi, grid, rcam).data, ref_img)
        img2, st2 = vb.render_vdi(gvdi, grid, rcam, with_stats=True)
        _, st1 = vb.render_vdi(vdi, grid, rcam, with_stats=True)
        assert np.array_equal(img2.data, ref_img)
        assert (st2.lists_visited, st2.supersegments_intersected, st2.lists_searched) == \
            (st1.lists_visited, st1.supersegments_intersected, st1.lists_searched)


def test_bricked_c3_four_ranks():
    _check("C3", 4)


def test_bricked_c3_four_ranks_balanced():
    """Contiguous bands of unequal height from the per-row executed samples
    (shard.balance_bands), each rank with only its box resident."""
    _check("C3", 4, balanced=True)


def test_bricked_c5_eight_ranks():
    _check("C5", 8, box_volume=lambda org, size: synth.rm_like(box=(org, size)).device_data,
           max_frac=0.4)
