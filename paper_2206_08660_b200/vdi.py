"""VDI and AccelGrid containers (mirror `pkg/src/vdikit/vdi.py:43-79`).

The reference types are frozen dataclasses of host numpy arrays:
  Vdi.counts (H, W) i32, Vdi.segs (H, W, n_sg, 6) f32 [front, back, r, g, b, a]
  AccelGrid.counts (gz, gy, gx) u32
Ours carry the same attributes and constructor, plus an optional device
residency: a VDI produced by `generate_vdi` stays on the GPU in the list-SoA
layout (include/vdi_b200.h) and `counts` / `segs` are materialised on first
access (one layout-conversion kernel + one pinned D2H copy). `render_vdi`
consumes the device copy directly, so generate -> render never round-trips
through the host; a host-only VDI (for instance a reference vdikit.Vdi) is
uploaded and converted once and the device copy is cached on the object.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _capi
from . import device as dv

F, B, R, G, BCH, A = 0, 1, 2, 3, 4, 5


class InvariantViolation(ValueError):
    pass


def default_grid_dims(width: int, height: int, gz: int = 32) -> tuple:
    """vdi.py:77-79: one cell per 16x16 lists, 32 depth slabs."""
    return (max(1, width // 16), max(1, height // 16), max(1, gz))


def ndc_z_to_view_depth(cam, ndc_z: float) -> float:
    n, f = cam.near, cam.far
    a = -(f + n) / (f - n)
    b = -2.0 * f * n / (f - n)
    return -b / (-ndc_z - a)


@dataclass
class DeviceVdi:
    """Device-resident lists: counts (rows, W) i32, segs (rows*W, n_sg*6) f32
    list-SoA. Storage rows may be band-interleaved after a multi-GPU
    all-gather (band_rows, world, rows_per_rank), see vdi_storage_row."""
    counts: object
    segs: object
    band_rows: int = 16
    world: int = 1
    rows_per_rank: int = 0
    # fronts and backs non-decreasing in every list: true of generated VDIs
    # (_emit clamps, generate.py:58-62); lets the render search before the
    # ESS test (VdiRenderArgs.lists_sorted)
    sorted: bool = False
    # storage row of every list row (device int32), overriding the band map:
    # the gathered VDI of contiguous bands of unequal height
    row_map: object = None


class Vdi:
    """Per-pixel supersegment lists of one generation viewpoint."""

    def __init__(self, width, height, n_sg, counts, segs, gen_camera, volume_aabb,
                 _device: DeviceVdi | None = None):
        self.width = int(width)
        self.height = int(height)
        self.n_sg = int(n_sg)
        self.gen_camera = gen_camera
        self.volume_aabb = np.asarray(volume_aabb, dtype=np.float64)
        self._counts = counts
        self._segs = segs
        self._device = _device

    # -- host views (materialised lazily from the device copy)
    @property
    def counts(self) -> np.ndarray:
        if self._counts is None:
            self._materialize()
        return self._counts

    @property
    def segs(self) -> np.ndarray:
        if self._segs is None:
            self._materialize()
        return self._segs

    def _materialize(self):
        t = dv.torch()
        d = self._device
        h, w, n = self.height, self.width, self.n_sg
        counts = d.counts
        segs = d.segs
        if d.world > 1:
            counts, segs = unshard_rows(d, h, w)
        aos = t.empty((h * w, n * 6), dtype=t.float32, device=segs.device)
        _capi.check(_capi.load().vdi_segs_to_aos(dv.ptr(segs), dv.ptr(aos), h * w, n,
                                                 dv.stream_handle()))
        self._counts = dv.to_host(counts[:h], sync=False)
        self._segs = dv.to_host(aos, sync=True).reshape(h, w, n, 6)

    def device(self) -> DeviceVdi:
        if self._device is None:
            t = dv.require_cuda()
            h, w, n = self.height, self.width, self.n_sg
            counts = dv.to_device(np.ascontiguousarray(self._counts, np.int32))
            aos = dv.to_device(np.ascontiguousarray(self._segs, np.float32).reshape(h * w, n * 6))
            soa = t.empty((h * w, (6 * n + 3) & ~3), dtype=t.float32, device="cuda")
            _capi.check(_capi.load().vdi_segs_from_aos(dv.ptr(aos), dv.ptr(soa), h * w, n,
                                                       dv.stream_handle()))
            self._device = DeviceVdi(counts=counts.view(h, w), segs=soa)
        return self._device

    def list_at(self, lx: int, ly: int) -> np.ndarray:
        return self.segs[ly, lx, : self.counts[ly, lx]]


def unshard_rows(d: DeviceVdi, h: int, w: int):
    """Band-interleaved storage rows -> natural row order (device gather)."""
    t = dv.torch()
    rows = np.arange(h)
    b = rows // d.band_rows
    store = (b % d.world) * d.rows_per_rank + (b // d.world) * d.band_rows + rows % d.band_rows
    idx = t.from_numpy(store).to(d.counts.device)
    counts = d.counts.index_select(0, idx)
    segs = d.segs.view(-1, w, d.segs.shape[1]).index_select(0, idx).reshape(h * w, -1)
    return counts, segs


class AccelGrid:
    """Per-cell supersegment counts over the frustum-aligned grid."""

    def __init__(self, dims, counts, near, far, _device=None):
        self.dims = tuple(int(v) for v in dims)
        self.near = float(near)
        self.far = float(far)
        self._counts = counts
        self._device = _device

    @property
    def counts(self) -> np.ndarray:
        if self._counts is None:
            self._counts = dv.to_host(self._device).view(np.uint32)
        return self._counts

    @property
    def z_slabs(self) -> np.ndarray:
        return np.linspace(self.near, self.far, self.dims[2] + 1)

    def device(self):
        if self._device is None:
            dv.require_cuda()
            self._device = dv.to_device(np.ascontiguousarray(self._counts, np.uint32).view(np.int32))
        return self._device


_VIOLATIONS = {1: "front >= back", 2: "overlapping supersegments",
               3: "depth outside [-1, 1]", 4: "color not premultiplied"}


def validate_vdi(vdi) -> None:
    """vdi.py:116-134 on the device (vdi_validate): raises the reference's
    InvariantViolation, with its message, for the count range or for the
    first violating list in row-major order."""
    from .raycast import _as_device_vdi
    t = dv.require_cuda()
    v = _as_device_vdi(vdi)
    d = v.device()
    res = t.empty(2, dtype=t.int64, device="cuda")
    a = _capi.VdiValidateArgs()
    a.segs, a.counts, a.result = dv.ptr(d.segs), dv.ptr(d.counts), dv.ptr(res)
    a.width, a.height, a.n_sg = v.width, v.height, v.n_sg
    a.vdi_band_rows, a.vdi_band_world, a.vdi_rows_per_rank = (int(d.band_rows), int(d.world),
                                                              int(d.rows_per_rank))
    _capi.check(_capi.load().vdi_validate(a, dv.stream_handle()))
    first, n_range = (int(x) for x in dv.to_host(res).view(np.uint64))
    if n_range:
        raise InvariantViolation("list count out of [0, n_sg]")
    if first != (1 << 64) - 1:
        lst, code = first >> 3, first & 7
        ly, lx = divmod(lst, v.width)
        raise InvariantViolation(f"list ({lx},{ly}): {_VIOLATIONS[code]}")


def grid_cell_of(ndc_pt, grid, cam):
    gx, gy, gz = grid.dims
    cx = min(max(int(math.floor((ndc_pt[0] + 1.0) * gx / 2.0)), 0), gx - 1)
    cy = min(max(int(math.floor((ndc_pt[1] + 1.0) * gy / 2.0)), 0), gy - 1)
    depth = ndc_z_to_view_depth(cam, float(ndc_pt[2]))
    cz = int(math.floor((depth - grid.near) / (grid.far - grid.near) * gz))
    return (cx, cy, min(max(cz, 0), gz - 1))
