"""C4 (BASELINE configs[3]) at full size against the oracle: Rayleigh-Taylor-
shaped 1024^3 f32, 1920x1080, n_sg 30. Generation on every ray; the novel-view
sweep 0-30 deg rendered on every pixel (RGBA + the three per-pixel
counters), the oracle rendering its own VDI and grid."""

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
def c4():
    vol, tf, gcam, rcam, n_sg = synth.config("C4")
    params = vb.GenParams(n_sg=n_sg)
    vdi, grid, st = vb.generate_vdi(vol, tf, gcam, params, with_stats=True)
    ref = ff.oracle_generate(vol, tf, gcam, params)
    pa, pb = oracle.depth_consts(gcam.near, gcam.far)
    rgrid = oracle.accumulate_grid(ref["counts"], ref["segs"], grid.dims, gcam.near, gcam.far,
                                   pa, pb)
    return vol, tf, gcam, params, vdi, grid, st, ref, rgrid


def test_c4_generation_every_ray(c4):
    vol, tf, gcam, params, vdi, grid, st, ref, rgrid = c4
    blk = parity.generation(ref, vdi.counts, vdi.segs, st.passes, st.samples, st.gammas)
    blk["grid_equal"] = bool(np.array_equal(grid.counts, rgrid))
    ff.record("C4/gen", blk)
    assert blk["ok"], blk
    assert blk["counts_equal_frac"] == 1.0 and blk["segs_bit_exact"], blk
    assert blk["passes_equal"] and blk["samples_equal"] and blk["gammas_bit_exact"], blk
    assert blk["grid_equal"]


@pytest.mark.parametrize("deg", [0.0, 5.0, 10.0, 15.0, 20.0, 25.0, 30.0])
def test_c4_render_sweep_every_pixel(c4, deg):
    vol, tf, gcam, params, vdi, grid, st, ref, rgrid = c4
    cam = synth.sweep_camera(vol, deg, gcam.viewport, radius_scale=1.6)
    img, lv, si, ls = ff.gpu_render(vdi, grid, cam)
    rr = ff.oracle_render(ref["counts"], ref["segs"], rgrid, vol, gcam, cam)
    blk = parity.render(rr, img, lv, si, ls)
    ff.record(f"C4/render{deg:g}", blk)
    assert blk["pixels"] == 1920 * 1080
    assert blk["ok"], blk
