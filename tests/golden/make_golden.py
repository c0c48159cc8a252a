"""Generate the golden parity fixtures from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports vdikit from /root/reference/pkg/src (numba JIT, writable
NUMBA_CACHE_DIR), runs R's own kernels on small deterministic scenes and writes
tests/golden/<case>.npz. Nothing at test time reads /root/reference: the
fixtures are the committed record of R's outputs.

Counters R does not expose (executed samples per ray, lists searched per
pixel) come from instrumented copies of generate.py / raycast.py built at run
time from R's source text: one counter line is inserted, everything else is
verbatim, and the instrumented outputs are asserted identical to R's.
"""

from __future__ import annotations

import math
import os
import re
import sys
import types

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import vdikit as vk  # noqa: E402
from vdikit import generate as rgen  # noqa: E402
from vdikit import raycast as rray  # noqa: E402

from paper_2206_08660_b200 import synth  # noqa: E402


# ------------------------------------------------------------ instrumentation

def _load_instrumented(modname, path, edits):
    src = open(path).read()
    src = src.replace("from ._geom", "from vdikit._geom")
    src = src.replace("from .camera", "from vdikit.camera")
    src = src.replace("from .vdi", "from vdikit.vdi")
    src = src.replace("from .volume", "from vdikit.volume")
    src = src.replace("from .image", "from vdikit.image")
    src = src.replace("cache=True", "cache=False")
    for old, new, count in edits:
        n = src.count(old)
        assert n == count, (modname, old, n)
        src = src.replace(old, new)
    mod = types.ModuleType(modname)
    mod.__file__ = path
    sys.modules[modname] = mod
    exec(compile(src, path, "exec"), mod.__dict__)
    return mod


def instrumented_generate():
    path = os.path.join(REF, "vdikit/generate.py")
    return _load_instrumented("gen_instr", path, [
        ("capped, out_seg, tseg):", "capped, out_seg, tseg, ctr):", 1),
        ("        if tb <= ta:\n            break\n",
         "        if tb <= ta:\n            break\n        ctr[0] += 1\n", 1),
        ("True, out_seg, tseg)", "True, out_seg, tseg, ctr)", 1),
        ("False, out_seg, tseg)", "False, out_seg, tseg, ctr)", 1),
        ("out_seg, tseg, high_seg):", "out_seg, tseg, high_seg, ctr):", 1),
        ("                                   out_seg, tseg, high_seg)",
         "                                   out_seg, tseg, high_seg, ctr[idx:idx + 1])", 1),
        ("counts, segs, gammas, passes):", "counts, segs, gammas, passes, ctr):", 1),
    ])


def instrumented_render():
    path = os.path.join(REF, "vdikit/raycast.py")
    return _load_instrumented("ray_instr", path, [
        ("early_term, bg, img, lists_vis, segs_int):",
         "early_term, bg, img, lists_vis, segs_int, srch):", 1),
        ("                if search:\n                    fronts",
         "                if search:\n                    srch[row, col] += 1\n"
         "                    fronts", 1),
    ])


GI = instrumented_generate()
RI = instrumented_render()


# ---------------------------------------------------------------- helpers

def r_volume(vol):
    """R Volume holding exactly the samples our Volume holds."""
    if vol.voxel_type == "f32":
        arr = np.ascontiguousarray(vol.data, np.float32)
        return vk.Volume(dims=vol.dims, voxel_type="u8", spacing=vol.spacing,
                         data=arr, value_range=vol.value_range, normalized=arr)
    return vk.make_volume(vol.data, vol.voxel_type, vol.spacing)


def r_camera(cam):
    return vk.Camera(position=tuple(float(v) for v in cam.position),
                     orientation=tuple(float(v) for v in cam.orientation),
                     fov_y=float(cam.fov_y), near=float(cam.near),
                     far=float(cam.far), viewport=tuple(int(v) for v in cam.viewport))


def cam_record(prefix, rcam):
    return {
        f"{prefix}_pose": np.array([*rcam.position, *rcam.orientation, rcam.fov_y,
                                    rcam.near, rcam.far], np.float64),
        f"{prefix}_viewport": np.array(rcam.viewport, np.int64),
        f"{prefix}_pv": rcam.proj_view(),
        f"{prefix}_inv_pv": rcam.inv_proj_view(),
    }


def pack_segs(counts, segs):
    """Valid supersegments only, in list order (the VDI1 packing)."""
    h, w = counts.shape
    mask = np.arange(segs.shape[2])[None, None, :] < counts[:, :, None]
    return segs[mask]


def run_generate(rvol, rtf, rcam, params):
    delta, step, lref = params.resolve(rvol)
    w, h = rcam.viewport
    counts = np.zeros((h, w), np.int32)
    segs = np.zeros((h, w, params.n_sg, 6), np.float32)
    gammas = np.zeros((h, w), np.float64)
    passes = np.zeros((h, w), np.int32)
    ctr = np.zeros(h * w, np.int64)
    aabb = rvol.aabb
    GI._generate_kernel(rvol.normalized, rtf.lut, rcam.proj_view(), rcam.inv_proj_view(),
                        *np.asarray(rcam.position, dtype=np.float64),
                        *aabb[0], *aabb[1], w, h, params.n_sg, delta, params.epsilon,
                        params.gamma_init, step, lref, counts, segs, gammas, passes, ctr)
    vdi, grid, st = vk.generate_vdi(rvol, rtf, rcam, params, with_stats=True)
    assert np.array_equal(vdi.counts, counts)
    assert np.array_equal(vdi.segs.view(np.uint32), segs.view(np.uint32))
    assert np.array_equal(st.gammas, gammas) and np.array_equal(st.passes, passes)
    return vdi, grid, st, ctr.reshape(h, w), (delta, step, lref)


def run_render(vdi, grid, rcam_new, opts):
    out_w, out_h = rcam_new.viewport
    img = np.zeros((out_h, out_w, 4), np.float64)
    lv = np.zeros((out_h, out_w), np.int64)
    si = np.zeros((out_h, out_w), np.int64)
    srch = np.zeros((out_h, out_w), np.int64)
    gen = vdi.gen_camera
    gx, gy, gz = grid.dims
    n, f = gen.near, gen.far
    pa = (f + n) / (f - n)
    pb = 2.0 * f * n / (f - n)
    RI._render_kernel(vdi.segs, vdi.counts, vdi.width, vdi.height, gen.proj_view(),
                      gen.inv_proj_view(), *vdi.volume_aabb[0], *vdi.volume_aabb[1],
                      rcam_new.inv_proj_view(),
                      *np.asarray(rcam_new.position, dtype=np.float64), out_w, out_h,
                      opts.use_ess, grid.counts, gx, gy, gz, grid.near, grid.far, pa, pb,
                      opts.early_term_alpha, np.asarray(opts.background, np.float64),
                      img, lv, si, srch)
    ref_img, st = vk.render_vdi(vdi, grid, rcam_new, opts, with_stats=True)
    assert np.array_equal(ref_img.data.view(np.uint64), img.view(np.uint64))
    assert st.lists_visited == lv.sum() and st.supersegments_intersected == si.sum()
    return img, lv, si, srch


def render_record(tag, rcam, opts, res):
    img, lv, si, srch = res
    rec = cam_record(tag, rcam)
    rec.update({
        f"{tag}_opts": np.array([float(opts.use_ess), opts.early_term_alpha,
                                 *opts.background], np.float64),
        f"{tag}_image": img, f"{tag}_lists_visited": lv.astype(np.int32),
        f"{tag}_segs_intersected": si.astype(np.int32),
        f"{tag}_lists_searched": srch.astype(np.int32),
    })
    return rec


def save(name, rec):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **rec)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def volume_case(name, vol, tf, gen_cam, render_specs, n_sg, delta=None, eps=1e-6,
                volume_from=None):
    rvol, rtf, rgc = r_volume(vol), vk.TransferFunction(tf.control_points), r_camera(gen_cam)
    assert np.array_equal(rtf.lut, tf.lut)
    params = vk.GenParams(n_sg=n_sg, delta=delta, epsilon=eps)
    vdi, grid, st, ctr, (dl, step, lref) = run_generate(rvol, rtf, rgc, params)
    rec = {
        "voxel_type": np.array(vol.voxel_type),
        "volume": vol.data if volume_from is None else np.zeros(0, vol.data.dtype),
        "volume_from": np.array(volume_from or ""),
        "volume_shape": np.array(vol.data.shape, np.int64),
        "spacing": np.array(vol.spacing, np.float64), "aabb": rvol.aabb,
        "lut": rtf.lut, "tf_points": np.array(tf.control_points, np.float64),
        "n_sg": np.array(n_sg), "delta": np.array(dl), "eps": np.array(params.epsilon),
        "gamma_init": np.array(params.gamma_init), "step": np.array(step),
        "lref": np.array(lref),
        "counts": vdi.counts, "segs_packed": pack_segs(vdi.counts, vdi.segs),
        "gammas": st.gammas, "passes": st.passes, "samples": ctr.astype(np.int32),
        "grid": grid.counts, "grid_dims": np.array(grid.dims, np.int64),
    }
    rec.update(cam_record("gen", rgc))
    for i, (cam, opts) in enumerate(render_specs):
        rc = r_camera(cam)
        rec.update(render_record(f"r{i}", rc, opts, run_render(vdi, grid, rc, opts)))
    rec["n_renders"] = np.array(len(render_specs))
    hist = np.bincount(st.passes.ravel(), minlength=23)
    print(f"{name}: hit rays {int((st.passes > 0).sum())}, passes hist {hist.tolist()}, "
          f"samples {int(ctr.sum())}, segs {int(vdi.counts.sum())}")
    save(name, rec)


def random_vdi_case(name, seeds):
    """The reference's A2 scenario (test_acceptance.py:104-119, conftest.py:92-125):
    invariant-respecting random VDIs rendered from random orbit views."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import random_vdi  # noqa: E402
    rec = {"seeds": np.array(seeds)}
    for s in seeds:
        rng = np.random.default_rng(s)
        vdi, grid = random_vdi(rng, width=32, height=32, n_sg=8)
        az = float(rng.uniform(0, 360))
        el = float(rng.uniform(-60, 60))
        cam = vk.orbit_camera((0.0, 0.0, 2.5), float(rng.uniform(3.0, 6.0)), az, el,
                              fov_y=0.8, near=0.3, far=25.0, viewport=(32, 32))
        t = f"s{s}"
        rec[f"{t}_counts"] = vdi.counts
        rec[f"{t}_segs"] = vdi.segs
        rec[f"{t}_grid"] = grid.counts
        rec[f"{t}_aabb"] = vdi.volume_aabb
        rec.update(cam_record(f"{t}_gen", vdi.gen_camera))
        for j, opts in enumerate((vk.RenderOptions(use_ess=True),
                                  vk.RenderOptions(use_ess=False),
                                  vk.RenderOptions(early_term_alpha=0.5,
                                                   background=(0.2, 0.3, 0.4, 0.7)))):
            rec.update(render_record(f"{t}_r{j}", cam, opts,
                                     run_render(vdi, grid, cam, opts)))
    save(name, rec)


def search_case(name, n_cases=20000):
    """find_first_supersegment vectors on a quantised grid that forces exact
    ties (test_acceptance.py:78-101) plus uniform queries."""
    rng = np.random.default_rng(1)
    grid = np.linspace(-1.0, 1.0, 17)
    n_max = 8
    fr = np.zeros((n_cases, n_max), np.float32)
    bk = np.zeros((n_cases, n_max), np.float32)
    cnt = np.zeros(n_cases, np.int32)
    de = np.zeros(n_cases, np.float64)
    dx = np.zeros(n_cases, np.float64)
    pp = np.zeros(n_cases, np.int32)
    oi = np.zeros(n_cases, np.int32)
    os_ = np.zeros(n_cases, np.int32)
    i = 0
    while i < n_cases:
        n = int(rng.integers(1, n_max + 1))
        vals = np.sort(rng.choice(grid, size=2 * n))
        if any(vals[2 * j] >= vals[2 * j + 1] for j in range(n)):
            continue
        segs = np.zeros((n, 6), np.float32)
        segs[:, 0] = vals[0::2]
        segs[:, 1] = vals[1::2]
        segs[:, 5] = 0.5
        for _ in range(min(25, n_cases - i)):
            if rng.random() < 0.5:
                d1, d2 = rng.choice(grid, size=2)
            else:
                d1, d2 = rng.uniform(-1.1, 1.1, size=2)
            p = int(rng.integers(-1, n + 1))
            idx, seed = vk.find_first_supersegment(segs, d1, d2, p=p)
            fr[i, :n] = segs[:, 0]
            bk[i, :n] = segs[:, 1]
            cnt[i], de[i], dx[i], pp[i] = n, d1, d2, p
            oi[i] = -1 if idx is None else idx
            os_[i] = seed
            i += 1
    save(name, dict(fronts=fr, backs=bk, counts=cnt, d_entry=de, d_exit=dx,
                    seeds=pp, index=oi, seed_out=os_))


def dvr_case(name, specs):
    """render_dvr (dvr.py:92-103) on the volumes of the generation fixtures.
    specs: (tag, volume fixture, our Volume, TF, camera, step, ref_step,
    early_term_alpha, background)."""
    rec = {"tags": np.array([s[0] for s in specs])}
    for tag, vfrom, vol, tf, cam, step, ref_step, et, bg in specs:
        rvol, rtf, rc = r_volume(vol), vk.TransferFunction(tf.control_points), r_camera(cam)
        img = vk.render_dvr(rvol, rtf, rc, step=step, ref_step=ref_step,
                            early_term_alpha=et, background=bg)
        rec.update(cam_record(tag, rc))
        rec[f"{tag}_volume_from"] = np.array(vfrom)
        rec[f"{tag}_lut"] = rtf.lut
        rec[f"{tag}_params"] = np.array([np.nan if step is None else step,
                                         np.nan if ref_step is None else ref_step, et,
                                         *bg], np.float64)
        rec[f"{tag}_image"] = img.data
        print(f"{name}/{tag}: alpha mean {img.data[..., 3].mean():.4f}")
    save(name, rec)


def dvr_main():
    vol, tf, gcam, rcam, _ = synth.config("C1")
    sph = synth.preset_volume("sphere", 64)
    stf = synth.preset_tf("sphere")
    scam = synth.sweep_camera(sph, 25.0, (96, 80), elevation_deg=10.0)
    bands = synth.preset_volume("bands", 64)
    bu16 = synth.make_volume(bands.data.astype(np.uint16) * 257 + 3, "u16")
    bview = synth.sweep_camera(bands, 50.0, (64, 64), elevation_deg=-20.0)
    z = np.arange(32)[:, None, None]
    stripes = np.broadcast_to(np.where(z % 6 < 3, 200, 0), (32, 32, 32)).astype(np.uint8)
    svol = synth.make_volume(stripes, "u8")
    stcam = synth.sweep_camera(svol, 30.0, (24, 24), elevation_deg=60.0)
    bg0 = (0.0, 0.0, 0.0, 1.0)
    dvr_case("dvr", [
        ("d0", "c1_blobs64", vol, tf, rcam, None, None, 0.999, bg0),
        ("d1", "c1_blobs64", vol, tf, gcam, 0.37, 0.5, 0.999, (0.2, 0.3, 0.4, 0.7)),
        ("d2", "sphere64_u8", sph, stf, scam, None, None, 0.5, bg0),
        ("d3", "bands64_u16_nsg4", bu16, synth.preset_tf("bands"), bview, 0.8, 0.6, 0.999,
         bg0),
        ("d4", "stripes32_capped", svol, stf, stcam, None, None, 1.0, (1.0, 1.0, 1.0, 0.5)),
    ])


def fixture_vdi(src):
    """A reference Vdi + AccelGrid rebuilt from a committed fixture:
    "<volume case>" or "random_vdi:<seed>"."""
    from golden_io import load, unpack_segs
    if src.startswith("random_vdi:"):
        g = load("random_vdi")
        t = "s" + src.split(":")[1]
        pose = g[f"{t}_gen_pose"]
        vp = g[f"{t}_gen_viewport"]
        counts, segs, aabb, grid = (g[f"{t}_counts"], g[f"{t}_segs"], g[f"{t}_aabb"],
                                    g[f"{t}_grid"])
    else:
        g = load(src)
        pose, vp = g["gen_pose"], g["gen_viewport"]
        counts, aabb, grid = g["counts"], g["aabb"], g["grid"]
        segs = unpack_segs(counts, g["segs_packed"], int(g["n_sg"]))
    cam = vk.Camera(position=tuple(pose[0:3]), orientation=tuple(pose[3:7]),
                    fov_y=float(pose[7]), near=float(pose[8]), far=float(pose[9]),
                    viewport=(int(vp[0]), int(vp[1])))
    h, w, n_sg, _ = segs.shape
    vdi = vk.Vdi(w, h, n_sg, counts, segs, cam, aabb)
    gz, gy, gx = grid.shape
    return vdi, vk.AccelGrid((gx, gy, gz), grid, cam.near, cam.far)


def preview_main():
    """render_preview (preview.py:233-268) on committed VDIs: low-res
    image, upsampled image, total and per-cell samples."""
    from vdikit.preview import PreviewParams, render_preview
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    vol, tf, gcam, rcam, _ = synth.config("C1")
    sph = synth.preset_volume("sphere", 64)
    sc = synth.sweep_camera(sph, 25.0, (128, 128), elevation_deg=10.0)
    bands = synth.preset_volume("bands", 64)
    bview = synth.sweep_camera(bands, 50.0, (64, 64), elevation_deg=-20.0)
    from vdikit import orbit_camera as r_orbit
    rv_cam = r_orbit((0.0, 0.0, 2.5), 4.0, 30.0, 20.0, fov_y=0.8, near=0.3, far=25.0,
                     viewport=(32, 32))
    specs = [
        ("p0", "c1_blobs64", r_camera(rcam), 1.0, 1.0, (128, 128), (0.0, 0.0, 0.0, 1.0)),
        ("p1", "c1_blobs64", r_camera(gcam), 0.5, 0.8, (128, 128), (0.2, 0.3, 0.4, 0.7)),
        ("p2", "sphere64_u8", r_camera(sc), 0.3, 0.5, (96, 64), (0.0, 0.0, 0.0, 1.0)),
        ("p3", "bands64_u16_nsg4", r_camera(bview), 0.7, 1.0, (64, 64), (1.0, 1.0, 1.0, 0.5)),
        ("p4", "random_vdi:0", rv_cam, 1.0, 0.25, (32, 32), (0.0, 0.0, 0.0, 1.0)),
        ("p5", "sphere64_u8", r_camera(sc), 1.0, 0.25, (128, 128), (0.0, 0.0, 0.0, 1.0)),
    ]
    rec = {"tags": np.array([s[0] for s in specs])}
    for tag, src, cam, d_i, d_r, disp, bg in specs:
        vdi, grid = fixture_vdi(src)
        params = PreviewParams(d_i=d_i, d_r=d_r, display=disp)
        img, st = render_preview(vdi, grid, cam, params, background=bg, with_stats=True)
        rec.update(cam_record(tag, cam))
        rec[f"{tag}_vdi_from"] = np.array(src)
        rec[f"{tag}_params"] = np.array([d_i, d_r, disp[0], disp[1], *bg], np.float64)
        rec[f"{tag}_image"] = img.data
        rec[f"{tag}_total_samples"] = np.array(st.total_samples, np.int64)
        rec[f"{tag}_cell_samples"] = st.cell_samples
        print(f"preview/{tag}: {st.total_samples} samples, image {img.data.shape}")
    save("preview", rec)


def lz4_inputs():
    """Byte strings for the LZ4 vectors: edge sizes around the 12-byte match
    limit and 5-byte literal tail, runs, periodic data, long literal runs,
    long matches (255-run length extensions) and random data."""
    rng = np.random.default_rng(11)
    out = [b"", b"a", b"abcdefghijkl", b"abcdefghijklm", b"\x00" * 13, b"\x00" * 1000,
           bytes(range(256)) * 40, rng.integers(0, 256, 5000, dtype=np.uint8).tobytes(),
           (b"VDI1" + bytes(rng.integers(0, 4, 3000, dtype=np.uint8))) * 3,
           rng.integers(0, 256, 300, dtype=np.uint8).tobytes() + b"\x07" * 70000 +
           rng.integers(0, 256, 17, dtype=np.uint8).tobytes()]
    words = [rng.integers(0, 256, int(k), dtype=np.uint8).tobytes()
             for k in rng.integers(3, 40, 60)]
    out.append(b"".join(words[int(i)] for i in rng.integers(0, 60, 4000)))
    return out


def codec_main():
    """encode_vdi (vdi.py:141-159) and lz4.compress (lz4.py:51-114, 171-175)
    on committed VDIs and byte vectors."""
    import hashlib
    from vdikit import lz4 as rlz4
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    rec = {}
    vdis = ["c1_blobs64", "sphere64_u8", "bands64_u16_nsg4", "blobs64_nsg3",
            "stripes32_capped", "random_vdi:0", "random_vdi:3"]
    rec["vdi_tags"] = np.array(vdis)
    for k, src in enumerate(vdis):
        vdi, grid = fixture_vdi(src)
        raw = vk.encode_vdi(vdi, grid)
        comp = rlz4.compress(raw)
        assert rlz4.decompress(comp, len(raw)) == raw
        v2, g2 = vk.decode_vdi(raw)
        assert vk.encode_vdi(v2, g2) == raw
        rec[f"v{k}_raw_sha256"] = np.array(hashlib.sha256(raw).hexdigest())
        rec[f"v{k}_raw_len"] = np.array(len(raw), np.int64)
        rec[f"v{k}_lz4"] = np.frombuffer(comp, np.uint8)
        print(f"codec/{src}: raw {len(raw)} B, lz4 {len(comp)} B")
    ins = lz4_inputs()
    rec["n_bytes_cases"] = np.array(len(ins))
    for k, b in enumerate(ins):
        comp = rlz4.compress(b)
        assert rlz4.decompress(comp, len(b)) == b
        rec[f"b{k}_in"] = np.frombuffer(b, np.uint8)
        rec[f"b{k}_lz4"] = np.frombuffer(comp, np.uint8)
    # validate_vdi (vdi.py:116-134): violation messages of the reference
    vdi0, _ = fixture_vdi("random_vdi:1")
    base_c = np.ascontiguousarray(vdi0.counts[:6, :8])
    base_s = np.ascontiguousarray(vdi0.segs[:6, :8])
    rng = np.random.default_rng(5)
    cases = []

    def nz_list():
        ys, xs = np.nonzero(base_c >= 2)
        k = int(rng.integers(0, len(ys)))
        return int(ys[k]), int(xs[k])

    cases.append((base_c.copy(), base_s.copy()))
    for kind in range(12):
        c, sg = base_c.copy(), base_s.copy()
        y, x = nz_list()
        if kind in (0, 6):
            sg[y, x, 0, 1] = sg[y, x, 0, 0]                       # front >= back
        elif kind in (1, 7):
            sg[y, x, 1, 0] = sg[y, x, 0, 1] - 1e-3                # overlap
        elif kind in (2, 8):
            sg[y, x, 0, 0] = -1.01                                # depth below -1
        elif kind == 3:
            sg[y, x, 1, 1] = 1.5                                  # depth above 1
        elif kind in (4, 9):
            sg[y, x, 0, 2] = sg[y, x, 0, 5] + 0.01                # not premultiplied
        elif kind == 5:
            c[y, x] = vdi0.n_sg + 1                               # count range
        elif kind == 10:                                          # two lists, two kinds
            y2, x2 = nz_list()
            sg[y, x, 0, 2] = sg[y, x, 0, 5] + 0.01
            sg[y2, x2, 1, 0] = sg[y2, x2, 0, 1] - 1e-3
        elif kind == 11:                                          # two checks in one list
            sg[y, x, 0, 2] = sg[y, x, 0, 5] + 0.01
            sg[y, x, 0, 0] = -1.5
        if kind >= 6:  # tie edges: exactly at the f32 tolerances
            if kind == 7:
                sg[y, x, 1, 0] = np.float32(sg[y, x, 0, 1]) - np.float32(1e-7)
            if kind == 8:
                sg[y, x, 0, 0] = np.float32(-1.0 - 1e-6)
        cases.append((c, sg))
    from vdikit import vdi as rvdi
    msgs = []
    for k, (c, sg) in enumerate(cases):
        v = vk.Vdi(8, 6, vdi0.n_sg, c, sg, vdi0.gen_camera, vdi0.volume_aabb)
        try:
            rvdi.validate_vdi(v)
            msgs.append("")
        except rvdi.InvariantViolation as e:
            msgs.append(str(e))
        rec[f"val{k}_counts"] = c
        rec[f"val{k}_segs"] = sg
    rec["val_messages"] = np.array(msgs)
    print("validate messages:", msgs)
    save("codec", rec)


def singles_main():
    """The reference's single-ray / test-facing functions: generate_list and
    find_gamma (generate.py:371-407) on pixel rays and off-axis rays of the C1
    scene, terminate_check (357-368), dda_traverse (raycast.py:225-234),
    project_ray_to_ndc (237-255) and composite_lists (494-518)."""
    from vdikit import generate as rg, raycast as rr
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    rvol, rtf, rc = r_volume(vol), vk.TransferFunction(tf.control_points), r_camera(gcam)
    rng = np.random.default_rng(21)
    rays = []
    for _ in range(96):
        px = (int(rng.integers(0, 128)), int(rng.integers(0, 128)))
        rays.append(vk.generate_ray(rc, px))
    for _ in range(32):  # off-axis rays from points around the volume
        o = np.asarray(rc.position) + rng.normal(0, 8, 3)
        tgt = rng.uniform(8, 56, 3)
        d = tgt - o
        rays.append(vk.Ray(origin=o, dir=d / np.linalg.norm(d)))
    rec = {"ray_o": np.array([r.origin for r in rays]), "ray_d": np.array([r.dir for r in rays])}
    gams = [1e-5, 0.01, 0.05, 0.2, 1.0]
    rec["gammas"] = np.array(gams)
    for pi, params in enumerate((vk.GenParams(n_sg=n_sg), vk.GenParams(n_sg=4, delta=1),
                                 vk.GenParams(n_sg=6, delta=0, epsilon=0.02))):
        rec[f"p{pi}"] = np.array([params.n_sg, -1 if params.delta is None else params.delta,
                                  params.epsilon])
        for gi, g in enumerate(gams):
            for cap in (0, 1):
                cn, sg, ex = [], [], []
                for r in rays:
                    c, sgl, e = rg.generate_list(r, rvol, rtf, g, params, rc, capped=bool(cap))
                    cn.append(c); sg.append(sgl.copy()); ex.append(e)
                rec[f"p{pi}_g{gi}_c{cap}_count"] = np.array(cn)
                rec[f"p{pi}_g{gi}_c{cap}_segs"] = np.array(sg)
                rec[f"p{pi}_g{gi}_c{cap}_exceeded"] = np.array(ex)
        fg, fn, fs, fp = [], [], [], []
        for r in rays:
            g, n, sgl, p = rg.find_gamma(r, rvol, rtf, params, rc)
            fg.append(g); fn.append(n); fs.append(sgl.copy()); fp.append(p)
        rec[f"p{pi}_fg_gamma"] = np.array(fg)
        rec[f"p{pi}_fg_count"] = np.array(fn)
        rec[f"p{pi}_fg_segs"] = np.array(fs)
        rec[f"p{pi}_fg_passes"] = np.array(fp)
    rec.update(cam_record("gen", rc))
    # terminate_check
    tc_in = rng.uniform(0, 1, (400, 9))
    tc_in[:, 7] = rng.uniform(0.2, 2.0, 400)       # step_len
    tc_in[:, 8] = rng.uniform(0.0, 0.8, 400)       # gamma
    rec["tc_in"] = tc_in
    rec["tc_out"] = np.array([rg.terminate_check(x[0:3], x[3], x[3:7], x[7], x[8])
                              for x in tc_in])
    # dda_traverse: random chords, axis-parallel and corner-tie chords
    grid = np.linspace(-1, 1, 9)
    chords = [rng.uniform(-1.1, 1.1, 6) for _ in range(150)]
    chords += [np.array([rng.choice(grid), rng.choice(grid), -0.5, rng.choice(grid),
                         rng.choice(grid), 0.5]) for _ in range(50)]
    chords += [np.array([0.1, -0.9, 0.0, 0.1, 0.9, 1.0]), np.array([-0.9, 0.3, 0, 0.9, 0.3, 0])]
    rec["dda_chords"] = np.array(chords)
    rec["dda_wh"] = np.array([[32, 24], [7, 5]])
    for wi, (w, h) in enumerate(((32, 24), (7, 5))):
        cells, zs, ns = [], [], []
        for ch in chords:
            out = rr.dda_traverse(ch[:3], ch[3:], w, h)
            ns.append(len(out))
            cells += [c for c, _, _ in out]
            zs += [(a, b) for _, a, b in out]
        rec[f"dda{wi}_n"] = np.array(ns)
        rec[f"dda{wi}_cells"] = np.array(cells)
        rec[f"dda{wi}_z"] = np.array(zs)
    # project_ray_to_ndc on the rays above, against the C1 generation camera
    prj, hit = [], []
    for r in rays:
        res = rr.project_ray_to_ndc(r, rc, rvol.aabb)
        hit.append(res is not None)
        prj.append(np.concatenate(res) if res is not None else np.zeros(6))
    rec["proj_hit"] = np.array(hit)
    rec["proj_out"] = np.array(prj)
    # composite_lists on committed VDIs
    for src, tag in (("random_vdi:0", "cl0"), ("sphere64_u8", "cl1")):
        vdi, _ = fixture_vdi(src)
        rec[f"{tag}_img"] = rr.composite_lists(vdi).data
        rec[f"{tag}_img_opts"] = rr.composite_lists(
            vdi, vk.RenderOptions(early_term_alpha=0.5, background=(0.2, 0.3, 0.4, 0.7))).data
    save("singles", rec)


def main():
    if "--only-singles" in sys.argv:
        singles_main()
        return
    if "--only-codec" in sys.argv:
        codec_main()
        return
    if "--only-dvr" in sys.argv:
        dvr_main()
        return
    if "--only-preview" in sys.argv:
        preview_main()
        return
    deg = math.radians
    RO = vk.RenderOptions
    # C1: the BASELINE config the CPU reference runs (blobs 64^3 f32, 128^2, n_sg 20)
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    c_el = synth.sweep_camera(vol, 25.0, (128, 128), elevation_deg=10.0)
    c_big = synth.sweep_camera(vol, 30.0, (160, 96))
    volume_case("c1_blobs64", vol, tf, gcam,
                [(rcam, RO()), (rcam, RO(use_ess=False)), (gcam, RO()),
                 (c_el, RO()), (c_big, RO(early_term_alpha=1.0))], n_sg)

    # R's own sphere fixture (conftest.py:33-39): u8 sphere 64^3, 128^2, n_sg 12
    sph = synth.preset_volume("sphere", 64)
    stf = synth.preset_tf("sphere")
    scam = synth.sweep_camera(sph, 0.0, (128, 128))
    center = (32.0, 32.0, 32.0)
    radius = float(np.linalg.norm(np.asarray(scam.position) - 32.0))
    from paper_2206_08660_b200.camera import orbit_camera
    s25 = orbit_camera(center, radius, 25.0, 10.0, fov_y=scam.fov_y, near=scam.near,
                       far=scam.far, viewport=scam.viewport)
    s30 = orbit_camera(center, radius, 30.0, 0.0, fov_y=scam.fov_y, near=scam.near,
                       far=scam.far, viewport=scam.viewport)
    volume_case("sphere64_u8", sph, stf, scam,
                [(scam, RO()), (s25, RO(use_ess=True)), (s25, RO(use_ess=False)),
                 (scam, RO(early_term_alpha=0.1)), (s30, RO())], 12)

    # bands at a tight budget: exercises aborted counting passes, epsilon
    # exits with the cached high segments, and capped passes
    bands = synth.preset_volume("bands", 64)
    bu16 = synth.make_volume(bands.data.astype(np.uint16) * 257 + 3, "u16")
    btf = synth.preset_tf("bands")
    bcam = synth.sweep_camera(bands, 20.0, (64, 64), elevation_deg=35.0)
    bview = synth.sweep_camera(bands, 50.0, (64, 64), elevation_deg=-20.0)
    volume_case("bands64_u16_nsg4", bu16, btf, bcam, [(bview, RO()), (bcam, RO())], 4,
                delta=1)
    volume_case("blobs64_nsg3", vol, tf, synth.sweep_camera(vol, 40.0, (48, 48)),
                [(synth.sweep_camera(vol, 70.0, (48, 48)), RO())], 3, delta=1,
                volume_from="c1_blobs64")
    # coarse epsilon + zero slack: most multi-pass rays leave through the
    # epsilon test and return the cached high-gamma segments
    volume_case("blobs64_eps", vol, tf, synth.sweep_camera(vol, 10.0, (40, 40)),
                [(synth.sweep_camera(vol, 35.0, (40, 40)), RO())], 5, delta=0,
                eps=0.02, volume_from="c1_blobs64")
    # more separated opaque layers than the budget: count > n_sg for every
    # gamma, so the bisection ends in the capped pass (generate.py:248-252)
    z = np.arange(32)[:, None, None]
    stripes = np.broadcast_to(np.where(z % 6 < 3, 200, 0), (32, 32, 32)).astype(np.uint8)
    svol = synth.make_volume(stripes, "u8")
    volume_case("stripes32_capped", svol, synth.preset_tf("sphere"),
                synth.sweep_camera(svol, 0.0, (24, 24), elevation_deg=80.0),
                [(synth.sweep_camera(svol, 30.0, (24, 24), elevation_deg=60.0), RO())], 3)

    random_vdi_case("random_vdi", [0, 1, 2, 3, 4, 5])
    search_case("search_fuzz")
    dvr_main()
    preview_main()
    codec_main()
    singles_main()


if __name__ == "__main__":
    main()
