"""The reference's acceptance criteria (pkg/tests/test_acceptance.py) run on
the device path: A2 ESS exactness, A4 generation budget + bisection, A6 codec
losslessness, A7 anisotropy trend, A8 quality trend, A9 preview budgeting.
(A1 is tests/test_gpu_parity.py's search fuzz, A3 tests/test_gpu_dvr.py, A5 a
property of the opacity formula and A10 the host PI controller,
tests/test_host_next.py; A11 is the TCP server, out of scope.) Scenes follow
the reference's conftest.py: sphere / bands 128^3 at 256x256, n_sg 12."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import codec, synth  # noqa: E402
from paper_2206_08660_b200.camera import Camera, generate_ray, look_at, orbit_camera  # noqa: E402
from paper_2206_08660_b200.generate import gen_rays  # noqa: E402
from paper_2206_08660_b200.preview import PreviewParams, render_preview  # noqa: E402
from paper_2206_08660_b200.vdi import default_grid_dims  # noqa: E402
from paper_2206_08660_b200.volume import grayscale_tf, make_volume  # noqa: E402
from oracle import oracle  # noqa: E402


def random_vdi(rng, width=32, height=32, n_sg=8, fill=0.6):
    """An invariant-respecting random VDI (the reference's conftest.py:92-125
    scenario) with its AccelGrid (oracle accumulate_grid)."""
    cam = Camera(position=(0.0, 0.0, 5.0), orientation=(0, 0, 0, 1), fov_y=0.8, near=1.0,
                 far=20.0, viewport=(width, height))
    counts = np.zeros((height, width), np.int32)
    segs = np.zeros((height, width, n_sg, 6), np.float32)
    for ly in range(height):
        for lx in range(width):
            if rng.random() > fill:
                continue
            n = int(rng.integers(1, n_sg + 1))
            edges = np.sort(rng.uniform(-1.0, 1.0, size=2 * n)).astype(np.float32)
            while np.any(np.diff(edges) <= 0):
                edges = np.sort(rng.uniform(-1, 1, size=2 * n)).astype(np.float32)
            counts[ly, lx] = n
            for k in range(n):
                a = rng.uniform(0.05, 1.0)
                rgb = rng.uniform(0.0, 1.0, size=3) * a
                segs[ly, lx, k] = [edges[2 * k], edges[2 * k + 1], *rgb, a]
    dims = default_grid_dims(width, height)
    pa, pb = oracle.depth_consts(cam.near, cam.far)
    grid = oracle.accumulate_grid(counts, segs, dims, cam.near, cam.far, pa, pb)
    aabb = np.array([[-2.0, -2.0, 1.0], [2.0, 2.0, 4.0]])
    return (vb.Vdi(width, height, n_sg, counts, segs, cam, aabb),
            vb.AccelGrid(dims, grid, cam.near, cam.far))


def _random_view(rng):
    az = float(rng.uniform(0, 360))
    el = float(rng.uniform(-60, 60))
    return orbit_camera((0.0, 0.0, 2.5), float(rng.uniform(3.0, 6.0)), az, el, fov_y=0.8,
                        near=0.3, far=25.0, viewport=(32, 32))


def _scene(preset):
    vol = synth.preset_volume(preset, 128)
    tf = synth.preset_tf(preset)
    cam = synth.sweep_camera(vol, 0.0, (256, 256))
    vdi, grid, st = vb.generate_vdi(vol, tf, cam, vb.GenParams(n_sg=12), with_stats=True)
    return vol, tf, cam, vdi, grid, st


@pytest.fixture(scope="module")
def sphere_vdi():
    return _scene("sphere")


@pytest.fixture(scope="module")
def bands_vdi():
    return _scene("bands")


def _deviated(cam, center, deg):
    radius = float(np.linalg.norm(np.asarray(cam.position) - center))
    return orbit_camera(tuple(center), radius, deg, 0.0, fov_y=cam.fov_y, near=cam.near,
                        far=cam.far, viewport=cam.viewport)


def ssim(a, b):
    """metrics.py:40-72 restated (test infrastructure): mean SSIM of the BT.709
    luma, 11x11 Gaussian window (sigma 1.5), border excluded."""
    from scipy.ndimage import gaussian_filter
    luma = np.array([0.2126, 0.7152, 0.0722])
    x = np.clip(a[..., :3], 0.0, 1.0) @ luma
    y = np.clip(b[..., :3], 0.0, 1.0) @ luma
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    f = lambda v: gaussian_filter(v, 1.5, truncate=3.5, mode="reflect")  # noqa: E731
    mx, my = f(x), f(y)
    vx, vy, cov = f(x * x) - mx * mx, f(y * y) - my * my, f(x * y) - mx * my
    s = ((2 * mx * my + c1) * (2 * cov + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))
    return float(np.mean(s[5:-5, 5:-5]))


def test_a2_ess_exactness():
    for seed in range(20):
        rng = np.random.default_rng(seed)
        vdi, grid = random_vdi(rng)
        cam = _random_view(rng)
        on = vb.render_vdi(vdi, grid, cam, vb.RenderOptions(use_ess=True)).data
        off = vb.render_vdi(vdi, grid, cam, vb.RenderOptions(use_ess=False)).data
        assert np.abs(on - off).max() <= 1e-6, seed


def test_a4_generation_budget_and_bisection(sphere_vdi):
    vol128, tf128, cam, vdi, grid, stats = sphere_vdi
    assert vdi.counts.max() <= vdi.n_sg
    assert stats.max_passes <= 22
    params = vb.GenParams(n_sg=10)
    empty = make_volume(np.zeros((16, 16, 16), dtype=np.uint8), "u8")
    ecam = look_at((8, 8, 48), (8, 8, 8), fov_y=0.6, near=10, far=100, viewport=(3, 3))
    eray = generate_ray(ecam, (1, 1))
    _, n, _, passes = vb.find_gamma(eray, empty, grayscale_tf(0.5), params, ecam)
    assert n == 0 and passes == 1
    solid = make_volume(np.full((16, 16, 16), 150, dtype=np.uint8), "u8")
    _, n, _, passes = vb.find_gamma(eray, solid, grayscale_tf(0.5), params, ecam)
    assert n == 1 and passes == 1
    # count(gamma) non-increasing over a 16-step ladder on 1000 random rays
    vol = synth.preset_volume("sphere", 64)
    tf = synth.preset_tf("sphere")
    cam64 = look_at((32, 32, 180), (32, 32, 32), fov_y=math.radians(35), near=40, far=400,
                    viewport=(32, 32))
    rng = np.random.default_rng(7)
    rays = [generate_ray(cam64, (int(rng.integers(0, 32)), int(rng.integers(0, 32))))
            for _ in range(1000)]
    prev = None
    for g in np.linspace(1e-5, math.sqrt(3.0), 16):
        c, _, _, _, _ = gen_rays(rays, vol, tf, params, cam64, 1, [float(g)] * len(rays))
        if prev is not None:
            assert np.all(c <= prev)
        prev = c


def test_a6_codec_losslessness():
    for seed in range(200):
        rng = np.random.default_rng(seed)
        vdi, grid = random_vdi(rng, width=6, height=6, n_sg=4)
        raw = codec.encode_vdi(vdi, grid)
        v2, g2 = codec.decode_vdi(raw)
        assert codec.encode_vdi(v2, g2) == raw, seed
        assert oracle.lz4_decompress(codec.compress(raw), len(raw)) == raw, seed


def test_a7_anisotropy_trend(sphere_vdi):
    vol, tf, cam, vdi, grid, _ = sphere_vdi
    center = np.asarray(vol.world_size) / 2.0
    visited = []
    for deg in (5, 10, 20, 40):
        _, st = vb.render_vdi(vdi, grid, _deviated(cam, center, deg), with_stats=True)
        visited.append(st.lists_visited)
        assert st.supersegments_intersected <= st.lists_visited
    assert all(a <= b for a, b in zip(visited, visited[1:]))


def test_a8_quality_trend(sphere_vdi, bands_vdi):
    scores = {}
    for name, (vol, tf, cam, vdi, grid, _) in (("sphere", sphere_vdi), ("bands", bands_vdi)):
        center = np.asarray(vol.world_size) / 2.0
        for deg in (5, 40):
            view = _deviated(cam, center, deg)
            img = vb.render_vdi(vdi, grid, view).data
            truth = vb.render_dvr(vol, tf, view).data
            scores[(name, deg)] = ssim(img, truth)
    assert scores[("sphere", 5)] > scores[("sphere", 40)]
    assert scores[("bands", 5)] > scores[("bands", 40)]
    assert scores[("sphere", 5)] >= 0.9


def test_a9_preview_budgeting(sphere_vdi):
    vol, tf, cam, vdi, grid, _ = sphere_vdi
    params = PreviewParams(d_i=0.5, d_r=0.8, display=cam.viewport)
    _, stats = render_preview(vdi, grid, cam, params, with_stats=True)
    assert np.all(stats.cell_samples[grid.counts == 0] == 0)
    totals = {}
    for d_r in (0.4, 0.8):
        _, s = render_preview(vdi, grid, cam, PreviewParams(d_i=0.5, d_r=d_r,
                                                            display=cam.viewport),
                              with_stats=True)
        totals[d_r] = s.total_samples
    assert totals[0.8] / totals[0.4] == pytest.approx(2.0, rel=0.2)
    full = vb.render_vdi(vdi, grid, cam).data
    exact = render_preview(vdi, grid, cam, PreviewParams(d_i=1.0, d_r=1.0,
                                                         display=cam.viewport)).data
    assert np.abs(exact - full).max() <= 0.02
