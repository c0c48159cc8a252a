"""The reference's single-ray and test-facing functions on the device
(vdi_gen_rays, vdi_dda_cells, vdi_project_rays, vdi_composite_lists) vs the
reference's own outputs (singles.npz, made by tests/golden/make_golden.py):
generate_list (counting and capped passes at 5 gammas) and find_gamma (3
parameter sets) on 96 pixel rays + 32 off-axis rays of the C1 scene,
dda_traverse on 202 chords (random, grid-aligned ties, axis-parallel) at two
grid sizes, project_ray_to_ndc on the same rays, composite_lists on two
committed VDIs. All bit for bit."""

import numpy as np
import pytest

import golden_io as gio

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import synth  # noqa: E402
from paper_2206_08660_b200.camera import Camera, Ray  # noqa: E402
from paper_2206_08660_b200.generate import gen_rays  # noqa: E402


@pytest.fixture(scope="module")
def scene():
    g = gio.load("singles")
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    cam = gio.camera(g, "gen")
    assert np.array_equal(cam.proj_view(), g["gen_pv"])
    rays = [Ray(origin=o, dir=d) for o, d in zip(g["ray_o"], g["ray_d"])]
    return g, vol, tf, cam, rays


def _params(g, pi):
    n_sg, delta, eps = g[f"p{pi}"]
    return vb.GenParams(n_sg=int(n_sg), delta=None if delta < 0 else int(delta),
                        epsilon=float(eps))


@pytest.mark.parametrize("pi", [0, 1, 2])
def test_generate_list_matches_reference(scene, pi):
    g, vol, tf, cam, rays = scene
    params = _params(g, pi)
    for gi, gam in enumerate(g["gammas"]):
        for cap in (0, 1):
            c, s, _, _, _ = gen_rays(rays, vol, tf, params, cam, 2 if cap else 1,
                                     [gam] * len(rays))
            key = f"p{pi}_g{gi}_c{cap}"
            assert np.array_equal(np.minimum(c, params.n_sg), g[f"{key}_count"]), key
            assert np.array_equal(c > params.n_sg, g[f"{key}_exceeded"]), key
            assert np.array_equal(s.view(np.uint32), g[f"{key}_segs"].view(np.uint32)), key
    n, s, e = vb.generate_list(rays[0], vol, tf, float(g["gammas"][2]), params, cam)
    assert n == g[f"p{pi}_g2_c0_count"][0] and e == g[f"p{pi}_g2_c0_exceeded"][0]


@pytest.mark.parametrize("pi", [0, 1, 2])
def test_find_gamma_matches_reference(scene, pi):
    g, vol, tf, cam, rays = scene
    params = _params(g, pi)
    c, s, gm, p, _ = gen_rays(rays, vol, tf, params, cam, 0)
    assert np.array_equal(c, g[f"p{pi}_fg_count"])
    assert np.array_equal(p, g[f"p{pi}_fg_passes"])
    assert np.array_equal(gm.view(np.uint64), g[f"p{pi}_fg_gamma"].view(np.uint64))
    ref = g[f"p{pi}_fg_segs"]
    for i in range(len(rays)):
        n = int(c[i])
        assert np.array_equal(s[i, :n].view(np.uint32), ref[i, :n].view(np.uint32)), i
    gam, n, segs, passes = vb.find_gamma(rays[5], vol, tf, params, cam)
    assert (n, passes) == (int(c[5]), int(p[5]))


def test_dda_traverse_matches_reference(scene):
    g = scene[0]
    for wi, (w, h) in enumerate(g["dda_wh"]):
        ns, cells, zs = g[f"dda{wi}_n"], g[f"dda{wi}_cells"], g[f"dda{wi}_z"]
        off = 0
        for q, ch in enumerate(g["dda_chords"]):
            out = vb.dda_traverse(ch[:3], ch[3:], int(w), int(h))
            assert len(out) == ns[q], q
            for j, (c, za, zb) in enumerate(out):
                assert c == tuple(cells[off + j]), (q, j)
                assert (za, zb) == tuple(zs[off + j]), (q, j)
            off += len(out)


def test_project_ray_to_ndc_matches_reference(scene):
    g, vol, tf, cam, rays = scene
    for i, r in enumerate(rays):
        res = vb.project_ray_to_ndc(r, cam, vol.aabb)
        assert (res is not None) == bool(g["proj_hit"][i]), i
        if res is not None:
            got = np.concatenate(res)
            assert np.array_equal(got.view(np.uint64), g["proj_out"][i].view(np.uint64)), i


def test_composite_lists_matches_reference():
    g = gio.load("singles")
    for src, tag in (("random_vdi:0", "cl0"), ("sphere64_u8", "cl1")):
        counts, segs, grid, gen, aabb = gio.fixture_vdi(src)
        p, vp = gen["gen_pose"], gen["gen_viewport"]
        cam = Camera(position=tuple(p[0:3]), orientation=tuple(p[3:7]), fov_y=float(p[7]),
                     near=float(p[8]), far=float(p[9]), viewport=(int(vp[0]), int(vp[1])))
        h, w, n_sg, _ = segs.shape
        vdi = vb.Vdi(w, h, n_sg, counts, segs, cam, aabb)
        img = vb.composite_lists(vdi).data
        assert np.array_equal(img.view(np.uint64), g[f"{tag}_img"].view(np.uint64)), tag
        img2 = vb.composite_lists(vdi, vb.RenderOptions(early_term_alpha=0.5,
                                                        background=(0.2, 0.3, 0.4, 0.7))).data
        assert np.array_equal(img2.view(np.uint64), g[f"{tag}_img_opts"].view(np.uint64)), tag
