"""Pin the CPU oracle (oracle/vdi_oracle.c) to the reference's own outputs.

Every fixture in tests/golden/ was produced by the reference (vdikit) itself;
the oracle must reproduce it bit for bit before it is trusted as the checker
of the B200 path.
"""

import numpy as np
import pytest

import golden_io as gio
from oracle import oracle


@pytest.mark.parametrize("case", gio.VOLUME_CASES)
def test_generate_bit_exact(case):
    g = gio.load(case)
    out = oracle.generate(gio.normalized(g), g["lut"], **gio.gen_inputs(g))
    assert np.array_equal(out["counts"], g["counts"])
    assert np.array_equal(out["segs"].view(np.uint32), gio.expected_segs(g).view(np.uint32))
    assert np.array_equal(out["gammas"].view(np.uint64), g["gammas"].view(np.uint64))
    assert np.array_equal(out["passes"], g["passes"])
    assert np.array_equal(out["samples"], g["samples"])


@pytest.mark.parametrize("case", gio.VOLUME_CASES)
def test_grid_bit_exact(case):
    g = gio.load(case)
    gc = gio.camera(g, "gen")
    pa, pb = oracle.depth_consts(gc.near, gc.far)
    grid = oracle.accumulate_grid(g["counts"], gio.expected_segs(g),
                                  tuple(g["grid_dims"]), gc.near, gc.far, pa, pb)
    assert np.array_equal(grid, g["grid"])


@pytest.mark.parametrize("case", gio.VOLUME_CASES)
def test_render_bit_exact(case):
    g = gio.load(case)
    gc = gio.camera(g, "gen")
    segs = gio.expected_segs(g)
    for spec in gio.render_specs(g):
        t = spec["tag"]
        out = oracle.render(segs, g["counts"], g["gen_pv"], g["gen_inv_pv"], g["aabb"],
                            spec["inv_pv"], spec["eye"], *spec["viewport"], g["grid"],
                            gc.near, gc.far, spec["use_ess"], spec["early_term"],
                            spec["bg"])
        assert np.array_equal(out["image"].view(np.uint64), g[f"{t}_image"].view(np.uint64)), t
        assert np.array_equal(out["lists_visited"], g[f"{t}_lists_visited"]), t
        assert np.array_equal(out["segs_intersected"], g[f"{t}_segs_intersected"]), t
        assert np.array_equal(out["lists_searched"], g[f"{t}_lists_searched"]), t


def test_render_random_vdis_bit_exact():
    g = gio.load("random_vdi")
    for s in g["seeds"]:
        t = f"s{s}"
        pose = g[f"{t}_gen_pose"]
        near, far = pose[8], pose[9]
        for j in range(3):
            r = f"{t}_r{j}"
            o = g[f"{r}_opts"]
            vp = g[f"{r}_viewport"]
            out = oracle.render(g[f"{t}_segs"], g[f"{t}_counts"], g[f"{t}_gen_pv"],
                                g[f"{t}_gen_inv_pv"], g[f"{t}_aabb"], g[f"{r}_inv_pv"],
                                g[f"{r}_pose"][:3], int(vp[0]), int(vp[1]), g[f"{t}_grid"],
                                near, far, bool(o[0]), float(o[1]), o[2:6])
            assert np.array_equal(out["image"].view(np.uint64),
                                  g[f"{r}_image"].view(np.uint64)), r
            assert np.array_equal(out["lists_visited"], g[f"{r}_lists_visited"]), r
            assert np.array_equal(out["segs_intersected"], g[f"{r}_segs_intersected"]), r


def test_search_fuzz_matches_reference():
    g = gio.load("search_fuzz")
    for i in range(len(g["counts"])):
        idx, seed = oracle.find_first(g["fronts"][i], g["backs"][i], g["counts"][i],
                                      g["d_entry"][i], g["d_exit"][i], g["seeds"][i])
        assert idx == g["index"][i], i
        assert seed == g["seed_out"][i], i


def test_camera_matrices_bit_exact():
    """Our host Camera yields R's exact proj_view / inv_proj_view bits."""
    for case in gio.VOLUME_CASES:
        g = gio.load(case)
        tags = ["gen"] + [s["tag"] for s in gio.render_specs(g)]
        for t in tags:
            cam = gio.camera(g, t)
            assert np.array_equal(cam.proj_view().view(np.uint64), g[f"{t}_pv"].view(np.uint64))
            assert np.array_equal(cam.inv_proj_view().view(np.uint64),
                                  g[f"{t}_inv_pv"].view(np.uint64))


def test_dvr_bit_exact():
    """render_dvr (dvr.py:21-103): the oracle reproduces R's image bits."""
    for s in gio.dvr_specs():
        img = oracle.dvr(gio.normalized(s["vg"]), s["lut"], s["pv"], s["inv_pv"], s["eye"],
                         s["aabb"], s["width"], s["height"], s["step"], s["lref"],
                         s["early_term"], s["bg"])
        assert np.array_equal(img.view(np.uint64), s["image"].view(np.uint64)), s["tag"]


def _low_camera(s):
    from paper_2206_08660_b200.camera import Camera
    p = s["pose"]
    w, h = s["display"]
    low = (max(1, round(w * s["d_i"])), max(1, round(h * s["d_i"])))
    return Camera(position=tuple(p[0:3]), orientation=tuple(p[3:7]), fov_y=float(p[7]),
                  near=float(p[8]), far=float(p[9]), viewport=low)


@pytest.mark.parametrize("spec", gio.preview_specs(), ids=lambda s: s["tag"])
def test_preview_bit_exact(spec):
    """render_preview (preview.py:49-268): low-res point-sampled render +
    bilinear upsample; image bits, total and per-cell samples."""
    s = spec
    cam = _low_camera(s)
    gen = s["gen"]
    img, total, cells = oracle.preview_lowres(
        s["segs"], s["counts"], gen["gen_pv"], gen["gen_inv_pv"], s["aabb"],
        cam.inv_proj_view(), np.asarray(cam.position), *cam.viewport, s["grid"],
        float(gen["gen_pose"][8]), float(gen["gen_pose"][9]), s["d_r"], 0.999, s["bg"])
    up = oracle.bilinear_upsample(img, *s["display"])
    assert total == s["total"]
    assert np.array_equal(cells, s["cells"])
    assert np.array_equal(up.view(np.uint64), s["image"].view(np.uint64))


def _cam_vals(gen):
    p = gen["gen_pose"]
    return tuple(float(v) for v in p[:10])


def test_encode_vdi_bytes_match_reference():
    """vdi.py:141-159: the oracle's VDI1 bytes hash to the reference's."""
    import hashlib
    g = gio.load("codec")
    for k, src in enumerate(str(t) for t in g["vdi_tags"]):
        counts, segs, grid, gen, aabb = gio.fixture_vdi(src)
        h, w, n_sg, _ = segs.shape
        raw = oracle.encode_vdi(w, h, n_sg, counts, segs, _cam_vals(gen), aabb, grid)
        assert len(raw) == int(g[f"v{k}_raw_len"]), src
        assert hashlib.sha256(raw).hexdigest() == str(g[f"v{k}_raw_sha256"]), src
        assert oracle.lz4_compress(raw) == g[f"v{k}_lz4"].tobytes(), src
        assert oracle.lz4_decompress(g[f"v{k}_lz4"].tobytes(), len(raw)) == raw, src


def test_lz4_bit_exact():
    """lz4.py:51-168: compress is the reference's block bit for bit and
    decompress inverts it."""
    g = gio.load("codec")
    for k in range(int(g["n_bytes_cases"])):
        src = g[f"b{k}_in"].tobytes()
        exp = g[f"b{k}_lz4"].tobytes()
        assert oracle.lz4_compress(src) == exp, k
        assert oracle.lz4_decompress(exp, len(src)) == src, k


def test_lz4_decompress_rejects_malformed():
    """lz4.py:139-166 failure paths."""
    raw = bytes(range(200)) * 5
    comp = oracle.lz4_compress(raw)
    for bad in (comp[:-1], comp + b"\x00", b"\x1f\x00\x00", b"\x10a\x00\x00"):
        with pytest.raises(ValueError):
            oracle.lz4_decompress(bad, len(raw))
    with pytest.raises(ValueError):
        oracle.lz4_decompress(b"\x01", 0)
