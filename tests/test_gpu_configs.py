"""Full-size BASELINE configs beyond C1-C3 (parity cases, not bench lines).

C4: Rayleigh-Taylor-shaped 1024^3 f32 volume, 1920x1080, n_sg 30, novel-view
render sweep 0-30 deg. Generation is checked on every list (invariants) and
against the oracle on a deterministic sample of rows; every render of the sweep
is checked against the oracle on sampled rows, per pixel (RGBA and the
lists-visited / supersegments-intersected / lists-searched counters).
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
from paper_2206_08660_b200.raycast import launch_render  # noqa: E402
from oracle import oracle  # noqa: E402

ROWS = np.array([0, 97, 260, 431, 539, 540, 702, 888, 1079])


@pytest.fixture(scope="module")
def c4():
    vol, tf, gcam, rcam, n_sg = synth.config("C4")
    params = vb.GenParams(n_sg=n_sg)
    vdi, grid, st = vb.generate_vdi(vol, tf, gcam, params, with_stats=True)
    return vol, tf, gcam, n_sg, params, vdi, grid, st


def test_c4_generation(c4):
    vol, tf, gcam, n_sg, params, vdi, grid, st = c4
    assert vdi.counts.max() <= n_sg and st.passes.max() <= 23
    vb.validate_vdi(vdi)
    delta, step, lref = params.resolve(vol)
    w, h = gcam.viewport
    ref = oracle.generate(vol.normalized, tf.lut, gcam.proj_view(), gcam.inv_proj_view(),
                          np.asarray(gcam.position), vol.aabb, w, h, n_sg, delta,
                          params.epsilon, params.gamma_init, step, lref, rows=ROWS)
    same = vdi.counts[ROWS] == ref["counts"][ROWS]
    assert same.mean() >= 0.999
    s_gpu, s_ref = vdi.segs[ROWS], ref["segs"][ROWS]
    valid = (np.arange(n_sg)[None, None, :] < ref["counts"][ROWS][:, :, None]) & same[:, :, None]
    assert np.abs(s_gpu[..., :2] - s_ref[..., :2])[valid].max() <= 1e-5
    assert np.abs(s_gpu[..., 2:] - s_ref[..., 2:])[valid].max() <= 1e-3
    assert np.array_equal(st.passes[ROWS], ref["passes"][ROWS])
    assert np.array_equal(st.samples[ROWS], ref["samples"][ROWS])


@pytest.mark.parametrize("deg", [0.0, 5.0, 10.0, 15.0, 20.0, 25.0, 30.0])
def test_c4_render_sweep(c4, deg):
    vol, tf, gcam, n_sg, params, vdi, grid, st = c4
    cam = synth.sweep_camera(vol, deg, gcam.viewport, radius_scale=1.6)
    ow, oh = cam.viewport
    t = dv.torch()
    image = t.empty((oh, ow, 4), dtype=t.float64, device="cuda")
    pp = [t.empty((oh, ow), dtype=t.int32, device="cuda") for _ in range(3)]
    launch_render(vdi, grid, cam, vb.RenderOptions(), image, per_pixel=pp)
    img = dv.to_host(image)
    lv, si, ls = (dv.to_host(x) for x in pp)
    ref = oracle.render(vdi.segs, vdi.counts, gcam.proj_view(), gcam.inv_proj_view(), vol.aabb,
                        cam.inv_proj_view(), np.asarray(cam.position), ow, oh, grid.counts,
                        gcam.near, gcam.far, rows=ROWS)
    assert np.abs(img[ROWS] - ref["image"][ROWS]).max() <= 1e-3
    assert np.array_equal(lv[ROWS], ref["lists_visited"][ROWS])
    assert np.array_equal(si[ROWS], ref["segs_intersected"][ROWS])
    assert np.array_equal(ls[ROWS], ref["lists_searched"][ROWS])


def test_c3_pipeline_masked_cells_match_public_api():
    """The bench pipeline builds corner records only for bricks the
    empty-space test can sample (vdi_volume_cells_masked); its VDI must equal
    the public generate_vdi's (full corner records) bit for bit."""
    from paper_2206_08660_b200 import shard
    vol, tf, gcam, rcam, n_sg = synth.config("C3")
    params = vb.GenParams(n_sg=n_sg)
    vdi, grid = vb.generate_vdi(vol, tf, gcam, params)
    pipe = shard.Pipeline(vol, tf, gcam, rcam, params)
    assert pipe.cells is not None
    pipe.step()
    d = vdi.device()
    assert torch.equal(pipe.bufs.counts, d.counts)
    assert torch.equal(pipe.bufs.segs, d.segs)
    assert torch.equal(pipe.bufs.grid, grid.device())
