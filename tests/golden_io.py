"""Load the committed golden fixtures (made from the reference by
tests/golden/make_golden.py) into plain inputs/expected outputs."""

from __future__ import annotations

import functools
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
VOLUME_CASES = ["c1_blobs64", "sphere64_u8", "bands64_u16_nsg4", "blobs64_nsg3",
                "blobs64_eps", "stripes32_capped"]
VOXEL_MAX = {"u8": np.float32(255.0), "u16": np.float32(65535.0)}


@functools.lru_cache(maxsize=None)
def load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


def unpack_segs(counts, packed, n_sg):
    h, w = counts.shape
    segs = np.zeros((h, w, n_sg, 6), np.float32)
    mask = np.arange(n_sg)[None, None, :] < counts[:, :, None]
    segs[mask] = packed
    return segs


def volume_data(g):
    src = str(g["volume_from"])
    data = load(src)["volume"] if src else g["volume"]
    return data.reshape(tuple(g["volume_shape"]))


def normalized(g):
    """What R samples: Volume.normalized (volume.py:48-50)."""
    data = volume_data(g)
    vt = str(g["voxel_type"])
    if vt == "f32":
        return np.ascontiguousarray(data, np.float32)
    return data.astype(np.float32) / VOXEL_MAX[vt]


def camera(g, prefix):
    """Our Camera rebuilt from the stored pose (bit-compared in tests)."""
    from paper_2206_08660_b200.camera import Camera
    p = g[f"{prefix}_pose"]
    vp = g[f"{prefix}_viewport"]
    return Camera(position=tuple(p[0:3]), orientation=tuple(p[3:7]), fov_y=float(p[7]),
                  near=float(p[8]), far=float(p[9]), viewport=(int(vp[0]), int(vp[1])))


def gen_inputs(g):
    vp = g["gen_viewport"]
    return dict(pv=g["gen_pv"], inv_pv=g["gen_inv_pv"], eye=g["gen_pose"][:3],
                aabb=g["aabb"], width=int(vp[0]), height=int(vp[1]),
                n_sg=int(g["n_sg"]), delta=int(g["delta"]), eps=float(g["eps"]),
                gamma_init=float(g["gamma_init"]), step=float(g["step"]),
                lref=float(g["lref"]))


def expected_segs(g):
    return unpack_segs(g["counts"], g["segs_packed"], int(g["n_sg"]))


def render_specs(g):
    out = []
    for i in range(int(g["n_renders"])):
        t = f"r{i}"
        o = g[f"{t}_opts"]
        out.append(dict(tag=t, inv_pv=g[f"{t}_inv_pv"], eye=g[f"{t}_pose"][:3],
                        viewport=tuple(int(v) for v in g[f"{t}_viewport"]),
                        use_ess=bool(o[0]), early_term=float(o[1]), bg=o[2:6]))
    return out


def dvr_specs():
    """The render_dvr cases of dvr.npz (dvr.py:92-103), with the volume they
    ran on and step / ref_step resolved as render_dvr does."""
    g = load("dvr")
    out = []
    for t in (str(x) for x in g["tags"]):
        vg = load(str(g[f"{t}_volume_from"]))
        p = g[f"{t}_params"]
        step = 0.5 * float(np.min(vg["spacing"])) if np.isnan(p[0]) else float(p[0])
        lref = step if np.isnan(p[1]) else float(p[1])
        vp = g[f"{t}_viewport"]
        out.append(dict(tag=t, vg=vg, lut=g[f"{t}_lut"], pv=g[f"{t}_pv"],
                        inv_pv=g[f"{t}_inv_pv"], eye=g[f"{t}_pose"][:3],
                        aabb=vg["aabb"], width=int(vp[0]), height=int(vp[1]),
                        step=step, lref=lref, early_term=float(p[2]), bg=p[3:7],
                        image=g[f"{t}_image"],
                        step_arg=None if np.isnan(p[0]) else float(p[0]),
                        ref_step_arg=None if np.isnan(p[1]) else float(p[1])))
    return out


def fixture_vdi(src):
    """(counts, segs AoS, grid, gen prefix record, aabb) of a committed VDI:
    "<volume case>" or "random_vdi:<seed>"."""
    if src.startswith("random_vdi:"):
        g = load("random_vdi")
        t = "s" + src.split(":")[1]
        rec = {k[len(t) + 1:]: v for k, v in g.items() if k.startswith(f"{t}_gen_")}
        return g[f"{t}_counts"], g[f"{t}_segs"], g[f"{t}_grid"], rec, g[f"{t}_aabb"]
    g = load(src)
    rec = {k: v for k, v in g.items() if k.startswith("gen_")}
    return g["counts"], expected_segs(g), g["grid"], rec, g["aabb"]


def preview_specs():
    """The render_preview cases of preview.npz (preview.py:233-268)."""
    g = load("preview")
    out = []
    for t in (str(x) for x in g["tags"]):
        p = g[f"{t}_params"]
        counts, segs, grid, gen, aabb = fixture_vdi(str(g[f"{t}_vdi_from"]))
        out.append(dict(tag=t, counts=counts, segs=segs, grid=grid, gen=gen, aabb=aabb,
                        d_i=float(p[0]), d_r=float(p[1]), display=(int(p[2]), int(p[3])),
                        bg=p[4:8], pose=g[f"{t}_pose"], viewport=g[f"{t}_viewport"],
                        image=g[f"{t}_image"], total=int(g[f"{t}_total_samples"]),
                        cells=g[f"{t}_cell_samples"]))
    return out
