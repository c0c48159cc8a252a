"""Host logic of the SURVEY 8(f) components (no GPU): the preview
controller and budgets (the reference's tests/test_preview.py cases), the
VDI1 header and FrameResult.decode against the oracle's encode_vdi, and the
bricked-volume box planner."""

import numpy as np
import pytest

import golden_io as gio
from oracle import oracle
from paper_2206_08660_b200 import shard, synth
from paper_2206_08660_b200.camera import Camera
from paper_2206_08660_b200.preview import (PiController, PreviewParams, low_res_viewport,
                                           pi_update, samples_in_cell)


def test_samples_in_cell_like_reference():
    assert samples_in_cell(0.7, 5.0, 0) == 0
    assert samples_in_cell(1.0, 2.0, 3) == 6
    assert samples_in_cell(0.5, 1.0, 1) == 1
    assert samples_in_cell(0.49, 1.0, 1) == 0
    assert samples_in_cell(0.5, 1.0, 3) == 2
    base = samples_in_cell(0.25, 8.0, 4)
    assert samples_in_cell(0.5, 8.0, 4) == 2 * base
    with pytest.raises(ValueError):
        samples_in_cell(-0.1, 1.0, 1)


def test_preview_params_validation_and_low_res():
    with pytest.raises(ValueError):
        PreviewParams(d_i=0.0)
    with pytest.raises(ValueError):
        PreviewParams(d_r=1.5)
    assert low_res_viewport(PreviewParams(d_i=0.3, display=(96, 64))) == (29, 19)
    assert low_res_viewport(PreviewParams(d_i=0.5, display=(5, 3))) == (2, 2)  # round half even
    assert low_res_viewport(PreviewParams(d_i=0.01, display=(10, 10))) == (1, 1)


def test_pi_controller_like_reference():
    ctrl = PiController()
    assert ctrl.update(200.0, 30) < 1.0
    assert PiController(d_i=0.5).update(5.0, 30) > 0.5
    ctrl = PiController()
    for _ in range(50):
        ctrl.update(10000.0, 60)
    assert ctrl.d_i == ctrl.bounds[0]
    for _ in range(200):
        ctrl.update(0.01, 10)
    assert ctrl.d_i == ctrl.bounds[1]
    with pytest.raises(ValueError):
        pi_update(PiController(), 0.0, 30)
    for fps in (20, 30, 60):
        c, ctrl = 50.0, PiController()
        frame = c * ctrl.d_i ** 2
        for _ in range(60):
            d = ctrl.update(frame, fps)
            frame = c * d * d
        if c * ctrl.bounds[1] ** 2 > 1000.0 / fps:
            assert frame == pytest.approx(1000.0 / fps, rel=0.05)


def _fixture_cam(gen):
    p, vp = gen["gen_pose"], gen["gen_viewport"]
    return Camera(position=tuple(p[0:3]), orientation=tuple(p[3:7]), fov_y=float(p[7]),
                  near=float(p[8]), far=float(p[9]), viewport=(int(vp[0]), int(vp[1])))


def test_vdi1_header_and_decode_match_oracle():
    from paper_2206_08660_b200.codec import vdi1_header
    from paper_2206_08660_b200.stream import FrameResult
    from paper_2206_08660_b200.vdi import AccelGrid, Vdi
    for src in ("sphere64_u8", "random_vdi:2"):
        counts, segs, grid, gen, aabb = gio.fixture_vdi(src)
        cam = _fixture_cam(gen)
        h, w, n_sg, _ = segs.shape
        gz, gy, gx = grid.shape
        raw = oracle.encode_vdi(w, h, n_sg, counts, segs, tuple(gen["gen_pose"][:10]), aabb, grid)
        hdr = vdi1_header(Vdi(w, h, n_sg, counts, segs, cam, aabb),
                          AccelGrid((gx, gy, gz), grid, cam.near, cam.far))
        assert raw[:160] == hdr
        r = FrameResult(index=0, counts=None, segs=None, grid=None, image=np.zeros((1, 1, 4)),
                        vdi1=np.frombuffer(raw, np.uint8))
        c2, s2, g2 = r.decode()
        assert np.array_equal(c2, counts) and np.array_equal(g2, grid)
        assert np.array_equal(s2.view(np.uint32), segs.view(np.uint32))


def test_band_volume_box_is_a_slab():
    """Elevation-0 orbit camera: a contiguous row band needs a y-slab only;
    the union over bands covers every voxel row the full view can touch."""
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    w, h = gcam.viewport
    full = shard.band_volume_box(vol, gcam, 0, h)
    boxes = [shard.band_volume_box(vol, gcam, r0, r0 + h // 4) for r0 in range(0, h, h // 4)]
    for org, size in boxes:
        assert org[1] % 8 == 0 and size[1] < vol.dims[1]
        assert org[0] == full[0][0] and size[0] == full[1][0]
    ys = set()
    for org, size in boxes:
        ys.update(range(org[1], org[1] + size[1]))
    assert ys >= set(range(full[0][1] + 2, full[0][1] + full[1][1] - 2))


def test_terminate_check_matches_reference():
    """generate.py:357-368 (host predicate) on the reference's 400 cases."""
    from paper_2206_08660_b200.generate import terminate_check
    g = gio.load("singles")
    got = [terminate_check(x[0:3], x[3], x[3:7], x[7], x[8]) for x in g["tc_in"]]
    assert np.array_equal(np.array(got), g["tc_out"])
