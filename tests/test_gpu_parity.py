"""B200 path vs the reference: golden fixtures (made by the reference itself)
and the pinned CPU oracle on larger configs. All calls go through the
product API -> ctypes -> libvdi_b200.so (include/vdi_b200.h).

Tolerances (BASELINE.json north_star): per-ray counts bit-exact on >= 99.9% of
rays (remainder only at gamma ties), depths within 1e-5, composited RGBA
within 1e-3. Where the arithmetic allows it the tests demand more (bit-exact
integer outputs and counters).
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
from paper_2206_08660_b200.volume import make_volume, TransferFunction  # noqa: E402
from oracle import oracle  # noqa: E402

COUNT_FRAC = 0.999
DEPTH_TOL = 1e-5
RGBA_TOL = 1e-3


def _volume(g):
    vt = str(g["voxel_type"])
    return make_volume(gio.volume_data(g), vt, tuple(g["spacing"]))


def _tf(g):
    tf = TransferFunction(tuple(tuple(p) for p in g["tf_points"]))
    assert np.array_equal(tf.lut, g["lut"])
    return tf


def compare_generation(exp_counts, exp_segs, counts, segs, label=""):
    """north_star gate + a report of bit-exactness."""
    same = counts == exp_counts
    frac = same.mean()
    assert frac >= COUNT_FRAC, f"{label}: counts equal on {frac:.5f}"
    n = exp_segs.shape[2]
    valid = (np.arange(n)[None, None, :] < exp_counts[:, :, None]) & same[:, :, None]
    if valid.any():
        dd = np.abs(segs[..., :2] - exp_segs[..., :2])[valid].max()
        dc = np.abs(segs[..., 2:] - exp_segs[..., 2:])[valid].max()
        assert dd <= DEPTH_TOL, f"{label}: depth diff {dd}"
        assert dc <= RGBA_TOL, f"{label}: colour diff {dc}"
    bit = np.array_equal(segs.view(np.uint32)[same], exp_segs.view(np.uint32)[same])
    return frac, bit


@pytest.mark.parametrize("case", gio.VOLUME_CASES)
def test_generate_matches_reference(case):
    g = gio.load(case)
    vol, tf = _volume(g), _tf(g)
    cam = gio.camera(g, "gen")
    params = vb.GenParams(n_sg=int(g["n_sg"]), delta=int(g["delta"]), epsilon=float(g["eps"]))
    vdi, grid, st = vb.generate_vdi(vol, tf, cam, params, with_stats=True)
    exp = gio.expected_segs(g)
    frac, bit = compare_generation(g["counts"], exp, vdi.counts, vdi.segs, case)
    # everything integer the reference computes must match exactly
    assert frac == 1.0, f"{case}: {np.sum(vdi.counts != g['counts'])} count mismatches"
    assert bit, f"{case}: segments not bit-identical"
    assert np.array_equal(st.passes, g["passes"])
    assert np.array_equal(st.samples, g["samples"])
    assert np.array_equal(st.gammas.view(np.uint64), g["gammas"].view(np.uint64))
    assert np.array_equal(grid.counts, g["grid"])
    vb.validate_vdi(vdi)


@pytest.mark.parametrize("case", gio.VOLUME_CASES)
def test_render_matches_reference(case):
    g = gio.load(case)
    gen_cam = gio.camera(g, "gen")
    vdi = vb.Vdi(width=int(g["gen_viewport"][0]), height=int(g["gen_viewport"][1]),
                 n_sg=int(g["n_sg"]), counts=g["counts"], segs=gio.expected_segs(g),
                 gen_camera=gen_cam, volume_aabb=g["aabb"])
    grid = vb.AccelGrid(tuple(g["grid_dims"]), g["grid"], gen_cam.near, gen_cam.far)
    for spec in gio.render_specs(g):
        t = spec["tag"]
        cam = gio.camera(g, t)
        opts = vb.RenderOptions(use_ess=spec["use_ess"], early_term_alpha=spec["early_term"],
                                background=tuple(spec["bg"]))
        img, st = vb.render_vdi(vdi, grid, cam, opts, with_stats=True)
        diff = np.abs(img.data - g[f"{t}_image"]).max()
        assert diff <= RGBA_TOL, f"{case}/{t}: rgba diff {diff}"
        assert st.lists_visited == int(g[f"{t}_lists_visited"].sum()), t
        assert st.supersegments_intersected == int(g[f"{t}_segs_intersected"].sum()), t
        assert st.lists_searched == int(g[f"{t}_lists_searched"].sum()), t
        assert diff <= 1e-12, f"{case}/{t}: rgba diff {diff} (expected ~bit-exact)"


def test_render_random_vdis_match_reference():
    g = gio.load("random_vdi")
    for s in g["seeds"]:
        t = f"s{s}"
        gen = gio.camera(g, f"{t}_gen")
        counts, segs = g[f"{t}_counts"], g[f"{t}_segs"]
        vdi = vb.Vdi(counts.shape[1], counts.shape[0], segs.shape[2], counts, segs, gen,
                     g[f"{t}_aabb"])
        grid = vb.AccelGrid(vb.default_grid_dims(counts.shape[1], counts.shape[0]),
                            g[f"{t}_grid"], gen.near, gen.far)
        for j in range(3):
            r = f"{t}_r{j}"
            o = g[f"{r}_opts"]
            opts = vb.RenderOptions(use_ess=bool(o[0]), early_term_alpha=float(o[1]),
                                    background=tuple(o[2:6]))
            img, st = vb.render_vdi(vdi, grid, gio.camera(g, r), opts, with_stats=True)
            assert np.abs(img.data - g[f"{r}_image"]).max() <= 1e-12, r
            assert st.lists_visited == int(g[f"{r}_lists_visited"].sum()), r
            assert st.supersegments_intersected == int(g[f"{r}_segs_intersected"].sum()), r


def test_search_fuzz_matches_reference():
    """A1 (test_acceptance.py:78-101): seeded search == reference on exact ties."""
    g = gio.load("search_fuzz")
    lists = np.zeros((len(g["counts"]), g["fronts"].shape[1], 6), np.float32)
    lists[..., 0] = g["fronts"]
    lists[..., 1] = g["backs"]
    idx, seed = vb.raycast.find_first_batch(lists, g["counts"], g["d_entry"], g["d_exit"],
                                            g["seeds"])
    assert np.array_equal(idx, g["index"])
    assert np.array_equal(seed, g["seed_out"])


def _oracle_generate(vol, tf, cam, n_sg, rows=None):
    params = vb.GenParams(n_sg=n_sg)
    delta, step, lref = params.resolve(vol)
    w, h = cam.viewport
    return oracle.generate(vol.normalized, tf.lut, cam.proj_view(), cam.inv_proj_view(),
                           np.asarray(cam.position), vol.aabb, w, h, n_sg, delta,
                           params.epsilon, params.gamma_init, step, lref, rows=rows)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_config_generate_and_render_vs_oracle(name):
    vol, tf, gcam, rcam, n_sg = synth.config(name)
    vdi, grid, st = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg), with_stats=True)
    ref = _oracle_generate(vol, tf, gcam, n_sg)
    frac, bit = compare_generation(ref["counts"], ref["segs"], vdi.counts, vdi.segs, name)
    assert frac == 1.0 and bit
    assert np.array_equal(st.samples, ref["samples"])
    pa, pb = oracle.depth_consts(gcam.near, gcam.far)
    rgrid = oracle.accumulate_grid(ref["counts"], ref["segs"], grid.dims, gcam.near, gcam.far,
                                   pa, pb)
    assert np.array_equal(grid.counts, rgrid)
    img, rs = vb.render_vdi(vdi, grid, rcam, with_stats=True)
    rr = oracle.render(ref["segs"], ref["counts"], gcam.proj_view(), gcam.inv_proj_view(),
                       vol.aabb, rcam.inv_proj_view(), np.asarray(rcam.position),
                       *rcam.viewport, rgrid, gcam.near, gcam.far)
    assert np.abs(img.data - rr["image"]).max() <= RGBA_TOL
    assert rs.lists_visited == rr["lists_visited"].sum()
    assert rs.supersegments_intersected == rr["segs_intersected"].sum()


def test_c3_full_size_properties_and_row_sample():
    """BASELINE config 3 at full size (1920x1080, 1024x1024x795 u8): invariants
    on every list + oracle parity on a deterministic sample of rows."""
    vol, tf, gcam, rcam, n_sg = synth.config("C3")
    vdi, grid, st = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg), with_stats=True)
    assert vdi.counts.max() <= n_sg and st.passes.max() <= 23
    vb.validate_vdi(vdi)
    rows = np.array([0, 131, 300, 433, 540, 541, 777, 1079])
    ref = _oracle_generate(vol, tf, gcam, n_sg, rows=rows)
    frac, bit = compare_generation(ref["counts"][rows], ref["segs"][rows], vdi.counts[rows],
                                   vdi.segs[rows], "C3")
    assert frac >= COUNT_FRAC
    # grid soundness: every populated list's cells are non-empty
    img, rs = vb.render_vdi(vdi, grid, rcam, with_stats=True)
    assert rs.lists_visited > 0 and rs.supersegments_intersected > 0
    assert np.all(np.isfinite(img.data)) and img.data[..., 3].max() <= 1 + 1e-9


@pytest.mark.parametrize("case", ["c1_blobs64", "bands64_u16_nsg4"])
def test_generate_with_minimal_workspace_defers_but_matches(case):
    """A cache too small for the overflowing rays forces the deferral rounds
    and the fused fallback kernel; results must not change."""
    from paper_2206_08660_b200 import device as dv
    from paper_2206_08660_b200.generate import alloc_gen, launch_generate
    g = gio.load(case)
    vol, tf = _volume(g), _tf(g)
    cam = gio.camera(g, "gen")
    params = vb.GenParams(n_sg=int(g["n_sg"]), delta=int(g["delta"]), epsilon=float(g["eps"]))
    w, h = cam.viewport
    dims = tuple(int(v) for v in g["grid_dims"])
    bufs = alloc_gen(w, h, params.n_sg, dims, stats=True)
    vd, vt = dv.upload_volume(vol)
    launch_generate(vd, vt, vol.dims, dv.upload_lut(tf.lut), cam, vol.aabb, params,
                    params.resolve(vol), bufs, dims, workspace_bytes="min")
    d = vb.vdi.DeviceVdi(bufs.counts, bufs.segs)
    vdi = vb.Vdi(w, h, params.n_sg, None, None, cam, vol.aabb, _device=d)
    assert np.array_equal(vdi.counts, g["counts"])
    assert np.array_equal(vdi.segs.view(np.uint32), gio.expected_segs(g).view(np.uint32))
    assert np.array_equal(dv.to_host(bufs.passes), g["passes"])
    assert np.array_equal(dv.to_host(bufs.samples), g["samples"])
    assert np.array_equal(dv.to_host(bufs.gammas).view(np.uint64), g["gammas"].view(np.uint64))


@pytest.mark.parametrize("vt,dims", [("u8", (45, 38, 51)), ("u8", (48, 38, 51)),
                                     ("u16", (45, 38, 51)), ("f32", (45, 38, 51))])
def test_cells_layout_matches_gather(vt, dims, monkeypatch):
    """Corner records (vdi_volume_cells) and plain gathers give identical
    VDIs, stats included, for every voxel type (odd dims: clamped borders;
    nx % 4 == 0: the u8 4-cell path)."""
    rng = np.random.default_rng(7)
    base = synth.blobs(64).data[:dims[2], :dims[1], :dims[0]]
    if vt == "u8":
        data = (base * 255).astype(np.uint8)
    elif vt == "u16":
        data = (base * 65535).astype(np.uint16) ^ rng.integers(0, 64, base.shape, dtype=np.uint16)
    else:
        data = np.ascontiguousarray(base, dtype=np.float32)
    vol = make_volume(data, vt)
    tf = synth.preset_tf("blobs")
    cam = synth.sweep_camera(vol, 20.0, (96, 80))
    out = {}
    from paper_2206_08660_b200.tuning import TUNING
    for flag in ("0", "1"):
        monkeypatch.setattr(TUNING, "cells", flag == "1")
        vdi, grid, st = vb.generate_vdi(vol, tf, cam, vb.GenParams(n_sg=12), with_stats=True)
        out[flag] = (vdi.counts, vdi.segs, grid.counts, st.passes, st.samples)
    assert out["0"][0].sum() > 0
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(np.asarray(a), np.asarray(b))
