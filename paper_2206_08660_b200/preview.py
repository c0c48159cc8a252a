"""Preview rendering with dynamic subsampling: drop-in for `vdikit.preview`
(preview.py:1-297).

The point-sampled preview kernel (preview.py:49-205) and the bilinear
upsample (208-223) run on the device (`vdi_preview_launch`,
`vdi_bilinear_upsample`, include/vdi_b200.h); the low-res frame never
leaves HBM before it is upsampled. The PI controller that picks d_i
(preview.py:271-297) is host control logic and stays in Python, as
SURVEY.md 8(f) prescribes.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np

from . import _capi
from . import device as dv
from .camera import Camera
from .generate import depth_consts, _mat
from .image import Image


@dataclass(frozen=True)
class PreviewParams:
    """preview.py:28-40."""
    d_i: float = 1.0                 # image-space resolution factor
    d_r: float = 1.0                 # along-ray sampling rate
    target_fps: float = 30.0
    display: tuple = (256, 256)

    def __post_init__(self):
        if not (0.0 < self.d_i <= 1.0):
            raise ValueError("d_i must be in (0, 1]")
        if not (0.0 < self.d_r <= 1.0):
            raise ValueError("d_r must be in (0, 1]")


def samples_in_cell(d_r: float, isect_len: float, count: int) -> int:
    """preview.py:42-46: round-half-up(d_r * length * count)."""
    if d_r < 0 or isect_len < 0 or count < 0:
        raise ValueError("inputs must be non-negative")
    return int(math.floor(d_r * isect_len * count + 0.5))


@dataclass(frozen=True)
class PreviewStats:
    """preview.py:226-230."""
    total_samples: int
    cell_samples: np.ndarray  # (gz, gy, gx) int64
    frame_ms: float


def low_res_viewport(params: PreviewParams) -> tuple:
    """preview.py:238-240 (Python round, half to even)."""
    disp_w, disp_h = params.display
    return max(1, round(disp_w * params.d_i)), max(1, round(disp_h * params.d_i))


def preview_args(dvdi, n_sg, vdi_w, vdi_h, gen_cam, aabb, grid_dev, grid_dims, grid_near,
                 grid_far, cam_low, d_r, early_term, background, image, workspace,
                 cell_samples=None, stat_sums=None) -> _capi.VdiPreviewArgs:
    a = _capi.VdiPreviewArgs()
    a.segs, a.counts, a.grid, a.image = (dv.ptr(dvdi.segs), dv.ptr(dvdi.counts),
                                         dv.ptr(grid_dev), dv.ptr(image))
    a.cell_samples, a.stat_sums, a.workspace = (dv.ptr(cell_samples), dv.ptr(stat_sums),
                                                dv.ptr(workspace))
    _capi.fill(a.gen_pv, _mat(gen_cam.proj_view()))
    _capi.fill(a.gen_inv_pv, _mat(gen_cam.inv_proj_view()))
    _capi.fill(a.new_inv_pv, _mat(cam_low.inv_proj_view()))
    _capi.fill(a.eye, np.asarray(cam_low.position, dtype=np.float64))
    _capi.fill(a.aabb, np.asarray(aabb, dtype=np.float64).reshape(6))
    _capi.fill(a.bg, np.asarray(background, dtype=np.float64).reshape(4))
    pa, pb = depth_consts(gen_cam.near, gen_cam.far)
    a.near, a.far, a.proj_a, a.proj_b = float(grid_near), float(grid_far), pa, pb
    a.d_r, a.early_term = float(d_r), float(early_term)
    a.vdi_w, a.vdi_h, a.n_sg = int(vdi_w), int(vdi_h), int(n_sg)
    a.gx, a.gy, a.gz = (int(v) for v in grid_dims)
    a.out_w, a.out_h = (int(v) for v in cam_low.viewport)
    a.vdi_band_rows, a.vdi_band_world = int(dvdi.band_rows), int(dvdi.world)
    a.vdi_rows_per_rank = int(dvdi.rows_per_rank)
    return a


def upsample_device(src, out_w: int, out_h: int):
    """bilinear_upsample of a device (h, w, c) f64 tensor; identity when the
    sizes match (preview.py:211-212 returns its input)."""
    t = dv.torch()
    h, w, ch = src.shape
    if (w, h) == (out_w, out_h):
        return src
    dst = t.empty((out_h, out_w, ch), dtype=t.float64, device=src.device)
    _capi.check(_capi.load().vdi_bilinear_upsample(dv.ptr(src), int(w), int(h), dv.ptr(dst),
                                                   int(out_w), int(out_h), int(ch),
                                                   dv.stream_handle()))
    return dst


def bilinear_upsample(arr, out_w: int, out_h: int):
    """preview.py:208-223 on the device. Returns `arr` itself when the sizes
    match, like the reference; a numpy input gives a numpy output."""
    if hasattr(arr, "data_ptr"):
        return upsample_device(arr.contiguous().to(dv.torch().float64), out_w, out_h)
    h, w = arr.shape[:2]
    if (w, h) == (out_w, out_h):
        return arr
    dv.require_cuda()
    a = np.asarray(arr, dtype=np.float64)
    squeeze = a.ndim == 2
    src = dv.to_device(np.ascontiguousarray(a[..., None] if squeeze else a))
    out = dv.to_host(upsample_device(src, out_w, out_h))
    return out[..., 0] if squeeze else out


def render_preview(vdi, grid, cam_new, params: PreviewParams,
                   background=(0.0, 0.0, 0.0, 1.0), with_stats: bool = False):
    """Point-sampled preview; returns the upsampled Image (and PreviewStats).

    Mirrors preview.py:233-268."""
    from .raycast import _as_device_grid, _as_device_vdi
    t = dv.require_cuda()
    vdi = _as_device_vdi(vdi)
    grid = _as_device_grid(grid)
    disp_w, disp_h = params.display
    low_w, low_h = low_res_viewport(params)
    cam_low = Camera(position=cam_new.position, orientation=cam_new.orientation,
                     fov_y=cam_new.fov_y, near=cam_new.near, far=cam_new.far,
                     viewport=(low_w, low_h))
    gx, gy, gz = grid.dims
    image = t.empty((low_h, low_w, 4), dtype=t.float64, device="cuda")
    ws = t.empty(_capi.PREVIEW_WORKSPACE_BYTES, dtype=t.uint8, device="cuda")
    cells = t.empty((gz, gy, gx), dtype=t.int64, device="cuda") if with_stats else None
    sums = t.zeros(1, dtype=t.int64, device="cuda") if with_stats else None
    t_start = time.perf_counter()
    a = preview_args(vdi.device(), vdi.n_sg, vdi.width, vdi.height, vdi.gen_camera,
                     vdi.volume_aabb, grid.device(), grid.dims, grid.near, grid.far, cam_low,
                     params.d_r, 0.999, background, image, ws, cells, sums)
    _capi.check(_capi.load().vdi_preview_launch(a, dv.stream_handle()))
    up = upsample_device(image, disp_w, disp_h)
    out = dv.to_host(up)
    ms = (time.perf_counter() - t_start) * 1000.0
    img = Image.from_array(out)
    if not with_stats:
        return img
    return img, PreviewStats(total_samples=int(dv.to_host(sums)[0]),
                             cell_samples=dv.to_host(cells), frame_ms=ms)


@dataclass
class PiController:
    """preview.py:271-282: holds d_i near a target frame rate; clamped
    output, anti-windup integral."""

    kp: float = 6e-3
    ki: float = 9e-4
    d_i: float = 1.0
    integral: float = 0.0
    bounds: tuple = (0.1, 1.0)

    def update(self, measured_frame_ms: float, target_fps: float) -> float:
        return pi_update(self, measured_frame_ms, target_fps)


def pi_update(ctrl: PiController, measured_frame_ms: float, target_fps: float) -> float:
    """preview.py:285-297: one controller step; mutates ctrl, returns d_i."""
    if measured_frame_ms <= 0:
        raise ValueError("measured_frame_ms must be > 0")
    lo, hi = ctrl.bounds
    error = 1000.0 / target_fps - measured_frame_ms
    ctrl.integral += error
    span = (hi - lo) / ctrl.ki if ctrl.ki > 0 else math.inf
    ctrl.integral = min(max(ctrl.integral, -span), span)
    d_i = ctrl.d_i + ctrl.kp * error + ctrl.ki * ctrl.integral
    ctrl.d_i = min(max(d_i, lo), hi)
    return ctrl.d_i
