"""Drop-in fidelity: objects shaped exactly like the reference's own (frozen
dataclasses with vdikit's attributes -- a Volume carrying the f32
`normalized` copy volume.py:48-50 builds, a Vdi / AccelGrid of numpy
arrays, its GenParams / RenderOptions -- and none of this package's extras:
no normalized_is_derived, no device()) go through generate_vdi /
render_vdi and reproduce the reference's golden outputs bit for bit.

Also: a reference Vdi whose arrays the caller mutates in place renders the
mutated lists (no device copy is cached on the caller's object).
"""

from dataclasses import dataclass, field, replace

import numpy as np
import pytest

import golden_io as gio

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402


@dataclass(frozen=True)
class RVolume:  # vdikit.volume.Volume (volume.py:30-60)
    dims: tuple
    voxel_type: str
    spacing: tuple
    data: np.ndarray
    value_range: tuple
    normalized: np.ndarray = field(repr=False, default=None)

    @property
    def world_size(self):
        return np.array(self.dims, np.float64) * np.array(self.spacing, np.float64)

    @property
    def aabb(self):
        return np.array([[0.0, 0.0, 0.0], self.world_size])


@dataclass(frozen=True)
class RTransferFunction:  # volume.py:125-147 (only the baked LUT is read)
    points: tuple
    lut: np.ndarray


@dataclass(frozen=True)
class RGenParams:  # generate.py:28-50
    n_sg: int = 12
    delta: int | None = None
    epsilon: float = 1e-6
    gamma_init: float = 1e-5
    step: float | None = None
    ref_step: float | None = None
    alpha_early: float = 0.999

    def resolve(self, vol):
        step = self.step if self.step is not None else 0.5 * min(vol.spacing)
        lref = self.ref_step if self.ref_step is not None else step
        delta = max(1, int(0.15 * self.n_sg)) if self.delta is None else self.delta
        delta = min(delta, self.n_sg - 1)
        if not (0 < self.epsilon < 1):
            raise ValueError("epsilon must be in (0, 1)")
        if self.n_sg < 1:
            raise ValueError("n_sg must be >= 1")
        return delta, step, lref


@dataclass(frozen=True)
class RVdi:  # vdi.py:43-59
    width: int
    height: int
    n_sg: int
    counts: np.ndarray
    segs: np.ndarray
    gen_camera: object
    volume_aabb: np.ndarray


@dataclass(frozen=True)
class RAccelGrid:  # vdi.py:62-74
    dims: tuple
    counts: np.ndarray
    near: float
    far: float


@dataclass(frozen=True)
class RRenderOptions:  # raycast.py:28-36
    use_ess: bool = True
    early_term_alpha: float = 0.999
    background: tuple = (0.0, 0.0, 0.0, 1.0)


def r_volume(g):
    vt = str(g["voxel_type"])
    data = gio.volume_data(g)
    nz, ny, nx = data.shape
    return RVolume(dims=(nx, ny, nz), voxel_type=vt, spacing=tuple(float(s) for s in g["spacing"]),
                   data=data, value_range=(float(data.min()), float(data.max())),
                   normalized=gio.normalized(g))


@pytest.mark.parametrize("case", ["sphere64_u8", "bands64_u16_nsg4", "c1_blobs64"])
def test_generate_reference_shaped_objects(case):
    g = gio.load(case)
    vol = r_volume(g)
    assert not hasattr(vol, "normalized_is_derived") and not hasattr(vol, "device")
    tf = RTransferFunction(points=tuple(tuple(p) for p in g["tf_points"]), lut=g["lut"])
    cam = gio.camera(g, "gen")
    params = RGenParams(n_sg=int(g["n_sg"]), delta=int(g["delta"]), epsilon=float(g["eps"]))
    vdi, grid, st = vb.generate_vdi(vol, tf, cam, params, with_stats=True)
    assert np.array_equal(vdi.counts, g["counts"])
    assert np.array_equal(vdi.segs.view(np.uint32), gio.expected_segs(g).view(np.uint32))
    assert np.array_equal(grid.counts, g["grid"])
    assert np.array_equal(st.passes, g["passes"])
    assert np.array_equal(st.gammas.view(np.uint64), g["gammas"].view(np.uint64))


@pytest.mark.parametrize("case", ["sphere64_u8", "c1_blobs64"])
def test_render_reference_shaped_vdi(case):
    g = gio.load(case)
    gen_cam = gio.camera(g, "gen")
    vdi = RVdi(width=int(g["gen_viewport"][0]), height=int(g["gen_viewport"][1]),
               n_sg=int(g["n_sg"]), counts=g["counts"].copy(), segs=gio.expected_segs(g),
               gen_camera=gen_cam, volume_aabb=g["aabb"])
    assert not hasattr(vdi, "device")
    grid = RAccelGrid(tuple(int(v) for v in g["grid_dims"]), g["grid"], gen_cam.near, gen_cam.far)
    for spec in gio.render_specs(g):
        t = spec["tag"]
        opts = RRenderOptions(use_ess=spec["use_ess"], early_term_alpha=spec["early_term"],
                              background=tuple(spec["bg"]))
        img, st = vb.render_vdi(vdi, grid, gio.camera(g, t), opts, with_stats=True)
        assert np.abs(img.data - g[f"{t}_image"]).max() <= 1e-12, t
        assert st.lists_visited == int(g[f"{t}_lists_visited"].sum()), t
        assert st.supersegments_intersected == int(g[f"{t}_segs_intersected"].sum()), t


def test_mutated_reference_vdi_is_not_rendered_stale():
    g = gio.load("sphere64_u8")
    gen_cam = gio.camera(g, "gen")
    counts = g["counts"].copy()
    vdi = RVdi(width=int(g["gen_viewport"][0]), height=int(g["gen_viewport"][1]),
               n_sg=int(g["n_sg"]), counts=counts, segs=gio.expected_segs(g),
               gen_camera=gen_cam, volume_aabb=g["aabb"])
    grid = RAccelGrid(tuple(int(v) for v in g["grid_dims"]), g["grid"], gen_cam.near, gen_cam.far)
    cam = gio.camera(g, "r0")
    before = vb.render_vdi(vdi, grid, cam).data
    counts[...] = 0  # the caller empties every list in place
    after = vb.render_vdi(vdi, grid, cam).data
    empty = vb.render_vdi(replace(vdi, counts=np.zeros_like(counts)), grid, cam).data
    assert not np.array_equal(before, after)
    assert np.array_equal(after, empty)
