"""C3 (BASELINE configs[2], the bench workload) at full size, every ray and
every pixel against the oracle: Kingsnake-shaped 1024x1024x795 u8,
1920x1080, n_sg 20, generate at 0 deg, render at 15 deg.

Generation: counts, supersegment bits, passes, executed samples and gamma
bits on all 2,073,600 rays, and the AccelGrid. Render: RGBA and the three
per-pixel counters on all 2,073,600 pixels, the oracle rendering its own VDI
and grid (an independent chain from the same inputs)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import fullframe as ff  # noqa: E402
import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import synth  # noqa: E402
from oracle import oracle, parity  # noqa: E402


@pytest.fixture(scope="module")
def c3():
    vol, tf, gcam, rcam, n_sg = synth.config("C3")
    params = vb.GenParams(n_sg=n_sg)
    vdi, grid, st = vb.generate_vdi(vol, tf, gcam, params, with_stats=True)
    ref = ff.oracle_generate(vol, tf, gcam, params)
    pa, pb = oracle.depth_consts(gcam.near, gcam.far)
    rgrid = oracle.accumulate_grid(ref["counts"], ref["segs"], grid.dims, gcam.near, gcam.far,
                                   pa, pb)
    return vol, tf, gcam, rcam, params, vdi, grid, st, ref, rgrid


def test_c3_generation_every_ray(c3):
    vol, tf, gcam, rcam, params, vdi, grid, st, ref, rgrid = c3
    blk = parity.generation(ref, vdi.counts, vdi.segs, st.passes, st.samples, st.gammas)
    blk["grid_equal"] = bool(np.array_equal(grid.counts, rgrid))
    ff.record("C3/gen", blk)
    assert blk["rays"] == 1920 * 1080
    assert blk["ok"], blk
    # what the design guarantees beyond the north_star gate: bit-exact
    assert blk["counts_equal_frac"] == 1.0 and blk["segs_bit_exact"], blk
    assert blk["passes_equal"] and blk["samples_equal"] and blk["gammas_bit_exact"], blk
    assert blk["grid_equal"]


def test_c3_render_every_pixel(c3):
    vol, tf, gcam, rcam, params, vdi, grid, st, ref, rgrid = c3
    img, lv, si, ls = ff.gpu_render(vdi, grid, rcam)
    rr = ff.oracle_render(ref["counts"], ref["segs"], rgrid, vol, gcam, rcam)
    blk = parity.render(rr, img, lv, si, ls)
    ff.record("C3/render15", blk)
    assert blk["pixels"] == 1920 * 1080
    assert blk["ok"], blk
    assert blk["lists_visited_total"] > 0 and blk["segs_intersected_total"] > 0


def test_c3_pipeline_masked_cells_match_public_api(c3):
    """The bench pipeline builds corner records only for bricks the
    empty-space test can sample (vdi_volume_cells_masked); its VDI must equal
    the public generate_vdi's (full corner records) bit for bit."""
    from paper_2206_08660_b200 import shard
    vol, tf, gcam, rcam, params, vdi, grid, st, ref, rgrid = c3
    pipe = shard.Pipeline(vol, tf, gcam, rcam, params)
    assert pipe.cells is not None
    pipe.step()
    d = vdi.device()
    assert torch.equal(pipe.bufs.counts, d.counts)
    assert torch.equal(pipe.bufs.segs, d.segs)
    assert torch.equal(pipe.bufs.grid, grid.device())
