"""render_preview on the B200 (vdi_preview_launch + vdi_bilinear_upsample)
vs the reference and the oracle.

Golden: preview.npz holds the reference's own render_preview outputs
(preview.py:233-268) on committed VDIs: the upsampled image, the total and
the per-cell planned samples, for d_i in {0.3, 0.5, 0.7, 1.0}, d_r in
{0.25, 0.5, 0.8, 1.0}, non-square displays and coloured backgrounds. The
sample budgets are integers and must match exactly; the image is held to
1e-12 (pow() in the per-sample opacity is the only non-bit-exact step).
Plus the reference's own preview tests (tests/test_preview.py) on the
device path, and C2 at full size against the oracle.
"""

import numpy as np
import pytest

import golden_io as gio

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import synth  # noqa: E402
from paper_2206_08660_b200.camera import Camera  # noqa: E402
from paper_2206_08660_b200.preview import PreviewParams, render_preview  # noqa: E402
from oracle import oracle  # noqa: E402

TIGHT = 1e-12


def _vdi(spec):
    gen = spec["gen"]
    p, vp = gen["gen_pose"], gen["gen_viewport"]
    cam = Camera(position=tuple(p[0:3]), orientation=tuple(p[3:7]), fov_y=float(p[7]),
                 near=float(p[8]), far=float(p[9]), viewport=(int(vp[0]), int(vp[1])))
    h, w, n_sg, _ = spec["segs"].shape
    gz, gy, gx = spec["grid"].shape
    vdi = vb.Vdi(w, h, n_sg, spec["counts"], spec["segs"], cam, spec["aabb"])
    grid = vb.AccelGrid((gx, gy, gz), spec["grid"], cam.near, cam.far)
    return vdi, grid


@pytest.mark.parametrize("spec", gio.preview_specs(), ids=lambda s: s["tag"])
def test_preview_matches_reference(spec):
    vdi, grid = _vdi(spec)
    p = spec["pose"]
    cam = Camera(position=tuple(p[0:3]), orientation=tuple(p[3:7]), fov_y=float(p[7]),
                 near=float(p[8]), far=float(p[9]),
                 viewport=tuple(int(v) for v in spec["viewport"]))
    params = PreviewParams(d_i=spec["d_i"], d_r=spec["d_r"], display=spec["display"])
    img, st = render_preview(vdi, grid, cam, params, background=tuple(spec["bg"]),
                             with_stats=True)
    assert st.total_samples == spec["total"]
    assert np.array_equal(st.cell_samples, spec["cells"])
    diff = float(np.abs(img.data - spec["image"]).max())
    assert diff <= TIGHT, f"{spec['tag']}: max |rgba diff| {diff}"


@pytest.fixture(scope="module")
def sphere_vdi_small():
    """The reference's conftest.py:33-39 scene."""
    vol = synth.preset_volume("sphere", 64)
    tf = synth.preset_tf("sphere")
    cam = synth.sweep_camera(vol, 0.0, (128, 128))
    vdi, grid = vb.generate_vdi(vol, tf, cam, vb.GenParams(n_sg=12))
    return vol, tf, cam, vdi, grid


def test_preview_full_resolution_close_to_reference(sphere_vdi_small):
    vol, tf, cam, vdi, grid = sphere_vdi_small
    img = render_preview(vdi, grid, cam, PreviewParams(d_i=1.0, d_r=1.0, display=cam.viewport))
    ref = vb.render_vdi(vdi, grid, cam)
    assert np.abs(img.data - ref.data).max() < 0.02


def test_preview_zero_count_cells_get_zero_samples(sphere_vdi_small):
    vol, tf, cam, vdi, grid = sphere_vdi_small
    params = PreviewParams(d_i=0.5, d_r=0.8, display=cam.viewport)
    img, stats = render_preview(vdi, grid, cam, params, with_stats=True)
    assert stats.total_samples > 0
    assert np.all(stats.cell_samples[grid.counts == 0] == 0)


def test_preview_sample_count_scales_with_d_r(sphere_vdi_small):
    vol, tf, cam, vdi, grid = sphere_vdi_small
    totals = []
    for d_r in (0.25, 0.5, 1.0):
        params = PreviewParams(d_i=0.5, d_r=d_r, display=cam.viewport)
        _, stats = render_preview(vdi, grid, cam, params, with_stats=True)
        totals.append(stats.total_samples)
    assert totals[0] < totals[1] < totals[2]
    assert totals[2] / totals[1] == pytest.approx(2.0, rel=0.25)


def test_preview_output_matches_display_size(sphere_vdi_small):
    vol, tf, cam, vdi, grid = sphere_vdi_small
    img = render_preview(vdi, grid, cam, PreviewParams(d_i=0.3, d_r=0.5, display=(96, 64)))
    assert (img.width, img.height) == (96, 64)


def test_upsample_matches_reference_expressions():
    rng = np.random.default_rng(3)
    for (h, w, oh, ow) in ((4, 4, 16, 16), (5, 7, 13, 3), (8, 8, 8, 8), (6, 5, 6, 11)):
        arr = rng.uniform(size=(h, w, 4))
        got = vb.bilinear_upsample(arr, ow, oh)
        exp = oracle.bilinear_upsample(arr, ow, oh)
        assert np.array_equal(np.asarray(got).view(np.uint64), exp.view(np.uint64))
    arr = rng.uniform(size=(6, 5, 4))
    assert vb.bilinear_upsample(arr, 5, 6) is arr


def test_preview_c2_vs_oracle():
    vol, tf, gcam, rcam, n_sg = synth.config("C2")
    vdi, grid = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg))
    params = PreviewParams(d_i=0.5, d_r=0.5, display=(512, 512))
    img, st = render_preview(vdi, grid, rcam, params, with_stats=True)
    low = Camera(position=rcam.position, orientation=rcam.orientation, fov_y=rcam.fov_y,
                 near=rcam.near, far=rcam.far, viewport=(256, 256))
    ref, total, cells = oracle.preview_lowres(
        vdi.segs, vdi.counts, gcam.proj_view(), gcam.inv_proj_view(), vol.aabb,
        low.inv_proj_view(), np.asarray(low.position), 256, 256, grid.counts, gcam.near,
        gcam.far, 0.5)
    up = oracle.bilinear_upsample(ref, 512, 512)
    assert st.total_samples == total
    assert np.array_equal(st.cell_samples, cells)
    assert float(np.abs(img.data - up).max()) <= 1e-3
