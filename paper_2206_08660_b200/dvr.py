"""Ground-truth direct volume rendering: drop-in for `vdikit.render_dvr`
(dvr.py:92-103).

Same signature, validation and return type. The emission-absorption raycast
(dvr.py:21-89) -- the generation ray, clip and sampler, front-to-back
compositing with early termination -- runs in `vdi_dvr_launch`
(include/vdi_b200.h) on the device volume generation already caches, so an
identity-view comparison against `render_vdi` isolates the representation
error exactly as the reference intends (dvr.py:1-6).
"""

from __future__ import annotations

import numpy as np

from . import _capi
from . import device as dv
from .generate import _mat
from .image import Image


def resolve_steps(vol, step, ref_step) -> tuple:
    """dvr.py:97-101: step defaults to half the finest spacing; ref_step to step."""
    if step is None:
        step = 0.5 * min(vol.spacing)
    if step <= 0:
        raise ValueError("step must be > 0")
    lref = ref_step if ref_step is not None else step
    return float(step), float(lref)


def dvr_args(vol_dev, voxel_type, dims, lut_dev, cam, aabb, step, lref, early_term,
             background, image, workspace, samples=None, stat_sums=None, bricks=None,
             ess_max=-1.0, cells=None, band=(16, 1, 0)) -> _capi.VdiDvrArgs:
    a = _capi.VdiDvrArgs()
    a.volume = dv.ptr(cells if cells is not None else vol_dev)
    a.lut = dv.ptr(lut_dev)
    a.brick_max = dv.ptr(bricks)
    a.ess_max = float(ess_max) if bricks is not None else -1.0
    a.brick_log2 = dv.BRICK_LOG2
    a.image, a.samples, a.stat_sums = dv.ptr(image), dv.ptr(samples), dv.ptr(stat_sums)
    a.workspace = dv.ptr(workspace)
    _capi.fill(a.pv, _mat(cam.proj_view()))
    _capi.fill(a.inv_pv, _mat(cam.inv_proj_view()))
    _capi.fill(a.eye, np.asarray(cam.position, dtype=np.float64))
    _capi.fill(a.aabb, np.asarray(aabb, dtype=np.float64).reshape(6))
    _capi.fill(a.bg, np.asarray(background, dtype=np.float64).reshape(4))
    a.step, a.lref, a.early_term = float(step), float(lref), float(early_term)
    a.voxel_type = _capi.VOXEL[voxel_type] | (_capi.VOXEL_CELLS if cells is not None else 0)
    a.nx, a.ny, a.nz = (int(v) for v in dims)
    a.lut_n = int(lut_dev.shape[0])
    a.width, a.height = (int(v) for v in cam.viewport)
    a.band_rows, a.band_stride, a.band_offset = (int(v) for v in band)
    return a


def launch_dvr(vol_dev, voxel_type, dims, lut_dev, cam, aabb, step, lref, early_term,
               background, image, workspace, samples=None, stat_sums=None, bricks=None,
               ess_max=-1.0, cells=None, band=(16, 1, 0), stream=None) -> None:
    """Enqueue one DVR frame on the current stream (no sync, no alloc)."""
    a = dvr_args(vol_dev, voxel_type, dims, lut_dev, cam, aabb, step, lref, early_term,
                 background, image, workspace, samples, stat_sums, bricks, ess_max, cells,
                 band)
    _capi.check(_capi.load().vdi_dvr_launch(a, dv.stream_handle() if stream is None
                                            else stream))


def render_dvr(vol, tf, cam, step: float | None = None, ref_step: float | None = None,
               early_term_alpha: float = 0.999, background=(0.0, 0.0, 0.0, 1.0),
               *, cache_volume: bool = True, samples_out: list | None = None) -> Image:
    """Front-to-back emission-absorption raycast of the classified volume.

    Mirrors dvr.py:92-103. `samples_out`, when a list, receives the per-pixel
    executed-sample counts (an (h, w) int32 array) -- a counter the reference
    does not expose, used for the algorithmic-bytes accounting."""
    step, lref = resolve_steps(vol, step, ref_step)
    t = dv.require_cuda()
    width, height = cam.viewport
    vol_dev, vt = dv.upload_volume(vol, cache=cache_volume)
    lut_dev = dv.upload_lut(tf.lut)
    bricks = dv.volume_bricks(vol_dev, vt, vol.dims)
    cells = dv.volume_cells(vol_dev, vt, vol.dims) if dv.use_cells(vt, vol.dims) else None
    image = t.empty((height, width, 4), dtype=t.float64, device="cuda")
    ws = t.empty(_capi.DVR_WORKSPACE_BYTES, dtype=t.uint8, device="cuda")
    samples = (t.empty((height, width), dtype=t.int32, device="cuda")
               if samples_out is not None else None)
    launch_dvr(vol_dev, vt, vol.dims, lut_dev, cam, np.asarray(vol.aabb, np.float64), step,
               lref, early_term_alpha, background, image, ws, samples=samples, bricks=bricks,
               ess_max=dv.ess_threshold(tf.lut), cells=cells)
    img = Image.from_array(dv.to_host(image))
    if samples_out is not None:
        samples_out.append(dv.to_host(samples))
    return img
