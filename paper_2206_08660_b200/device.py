"""Device plumbing: torch owns device memory and streams; the compute is in
libvdi_b200.so. Host<->device traffic goes through pinned staging buffers.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _capi

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise _capi.VdiError("paper_2206_08660_b200 needs a CUDA device (B200); "
                             "there is no CPU fallback")
    _capi.load()
    return t


def stream_handle():
    return torch().cuda.current_stream().cuda_stream


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def pinned_empty(shape, dtype):
    t = torch()
    return t.empty(shape, dtype=dtype, pin_memory=True)


def to_device(arr: np.ndarray, dtype=None):
    """H2D copy; pinned arrays (see pinned_numpy) copy asynchronously."""
    t = torch()
    a = np.ascontiguousarray(arr if dtype is None else arr.astype(dtype, copy=False))
    import warnings
    with warnings.catch_warnings():
        # read-only sources (bytes objects) are only read by the copy
        warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
        return t.from_numpy(a).to("cuda", non_blocking=True)


def pinned_numpy(shape, np_dtype) -> np.ndarray:
    """A numpy array backed by pinned host memory."""
    t = torch()
    if not _TORCH_OF:
        _init_dtypes()
    tt = t.empty(tuple(shape), dtype=_TORCH_OF[np.dtype(np_dtype)], pin_memory=True)
    return tt.numpy()


def to_host(dev_tensor, sync: bool = True) -> np.ndarray:
    """D2H through a pinned staging buffer."""
    host = torch().empty(dev_tensor.shape, dtype=dev_tensor.dtype, pin_memory=True)
    host.copy_(dev_tensor, non_blocking=True)
    if sync:
        torch().cuda.current_stream().synchronize()
    return host.numpy()


_TORCH_OF = {}


def _init_dtypes():
    t = torch()
    _TORCH_OF.update({np.dtype(np.uint8): t.uint8, np.dtype(np.int16): t.int16,
                      np.dtype(np.uint16): t.uint16, np.dtype(np.int32): t.int32,
                      np.dtype(np.uint32): t.uint32, np.dtype(np.int64): t.int64,
                      np.dtype(np.float32): t.float32, np.dtype(np.float64): t.float64})


class _ArrayCache:
    """Device copies of immutable host arrays (Volume.data, TF LUTs), keyed by
    identity and validated through a weak reference."""

    def __init__(self, capacity: int = 4):
        self.capacity = capacity
        self.items = []  # (weakref, key, tensor)

    def get(self, arr: np.ndarray, dtype=None):
        key = (arr.ctypes.data, arr.shape, arr.dtype.str)
        for i, (ref, k, tens) in enumerate(self.items):
            if k == key and ref() is arr:
                self.items.append(self.items.pop(i))
                return tens
        tens = to_device(arr, dtype)
        self.items.append((weakref.ref(arr), key, tens))
        while len(self.items) > self.capacity:
            self.items.pop(0)
        return tens

    def clear(self):
        self.items.clear()


volume_cache = _ArrayCache(2)
lut_cache = _ArrayCache(8)


def volume_array(vol):
    """(host array, voxel type) the device samples for `vol`.

    Our Volume with a derived `normalized` uploads the raw u8/u16 brick
    (normalised on the fly, bit-identical to volume.py:48-50); anything else
    (a reference vdikit.Volume, or a user-supplied `normalized`) uploads the
    f32 array the reference samples."""
    derived = getattr(vol, "normalized_is_derived", False)
    vt = getattr(vol, "voxel_type", "u8")
    if derived and vt in ("u8", "u16", "f32"):
        return vol.data, vt
    return np.ascontiguousarray(vol.normalized, dtype=np.float32), "f32"


def upload_volume(vol, cache: bool = True):
    if hasattr(vol, "device_data"):  # DeviceVolume: already resident
        return vol.device_data, vol.voxel_type
    arr, vt = volume_array(vol)
    if arr.ndim != 3:
        nx, ny, nz = vol.dims
        arr = arr.reshape(nz, ny, nx)
    if cache:
        return volume_cache.get(arr), vt
    return to_device(arr), vt


BRICK_LOG2 = 3
_bricks = {}


def volume_bricks(vol_dev, voxel_type: str, dims, log2: int = BRICK_LOG2):
    """Per-brick voxel maxima of a device volume (vdi_volume_brick_max), cached
    for as long as the device volume lives."""
    key = (vol_dev.data_ptr(), tuple(dims), voxel_type, log2)
    hit = _bricks.get(key)
    if hit is not None and hit[0]() is vol_dev:
        return hit[1]
    out = alloc_bricks(vol_dev, dims, log2)
    launch_bricks(vol_dev, voxel_type, dims, out, log2)
    for k in [k for k, v in _bricks.items() if v[0]() is None]:
        del _bricks[k]
    _bricks[key] = (weakref.ref(vol_dev), out)
    return out


def cells_bytes(voxel_type: str, dims) -> int:
    nx, ny, nz = (int(v) for v in dims)
    return int(_capi.load().vdi_volume_cells_bytes(_capi.VOXEL[voxel_type], nx, ny, nz))


def use_cells(voxel_type: str, dims) -> bool:
    """Whether generation samples from corner records (vdi_volume_cells): 8x
    the volume's bytes in exchange for one load per sample instead of 8
    gathers. tuning.TUNING.cells forces it. By default only u8 volumes use
    them (C3: build 1.8 ms, generation -2.5 ms; for f32, C4: build 9.6 ms for
    -3 ms), and only while the records fit in a quarter of device memory."""
    from .tuning import TUNING
    if TUNING.cells is not None:
        return bool(TUNING.cells)
    if voxel_type != "u8":
        return False
    total = torch().cuda.get_device_properties(torch().cuda.current_device()).total_memory
    return cells_bytes(voxel_type, dims) <= total // 4


def alloc_cells(voxel_type: str, dims):
    return torch().empty(cells_bytes(voxel_type, dims), dtype=torch().uint8, device="cuda")


def launch_cells(vol_dev, voxel_type: str, dims, out, bricks=None, ess_max=-1.0) -> None:
    """Corner records; with brick maxima and an ESS threshold, the records of
    bricks the samplers always skip are not written (vdi_volume_cells_masked)."""
    nx, ny, nz = (int(v) for v in dims)
    if bricks is not None and ess_max >= 0.0:
        _capi.check(_capi.load().vdi_volume_cells_masked(
            ptr(vol_dev), _capi.VOXEL[voxel_type], nx, ny, nz, ptr(bricks), BRICK_LOG2,
            float(ess_max), ptr(out), stream_handle()))
        return
    _capi.check(_capi.load().vdi_volume_cells(ptr(vol_dev), _capi.VOXEL[voxel_type], nx, ny, nz,
                                              ptr(out), stream_handle()))


def launch_bricks(vol_dev, voxel_type: str, dims, out, log2: int = BRICK_LOG2) -> None:
    nx, ny, nz = (int(v) for v in dims)
    _capi.check(_capi.load().vdi_volume_brick_max(ptr(vol_dev), _capi.VOXEL[voxel_type], nx, ny,
                                                   nz, log2, ptr(out), stream_handle()))


def alloc_bricks(vol_dev, dims, log2: int = BRICK_LOG2):
    nx, ny, nz = (int(v) for v in dims)
    b = 1 << log2
    return torch().empty(((nz + b - 1) // b, (ny + b - 1) // b, (nx + b - 1) // b),
                         dtype=vol_dev.dtype, device=vol_dev.device)


_cells = {}


def volume_cells(vol_dev, voxel_type: str, dims):
    """Corner records of a device volume, cached for as long as it lives. A
    new volume of the same shape (a new timestep, or an uncached upload)
    rebuilds into the previous buffer instead of allocating another
    8 x volume-sized block."""
    key = (tuple(dims), voxel_type)
    hit = _cells.get(key)
    if hit is not None and hit[0]() is vol_dev and hit[2] == vol_dev.data_ptr():
        return hit[1]
    out = hit[1] if hit is not None else alloc_cells(voxel_type, dims)
    for k in [k for k in _cells if k != key]:
        del _cells[k]
    launch_cells(vol_dev, voxel_type, dims, out)
    _cells[key] = (weakref.ref(vol_dev), out, vol_dev.data_ptr())
    return out


def ess_threshold(lut: np.ndarray) -> float:
    """Largest normalised brick maximum that guarantees alpha == 0.

    _lut_classify (volume.py:164-177) lerps rows i = floor(x), i + 1 with
    x = s (n - 1); if rows 0..K all have alpha 0, every s with x <= K
    classifies to alpha 0 exactly (x == K gives f == 0). A 1e-6 margin in x
    covers the few-ulp overshoot of a trilinear mix over its inputs. Returns
    -1 (no skipping) when row 0 is already visible."""
    a = np.asarray(lut, dtype=np.float32)[:, 3]
    n = len(a)
    nz = np.nonzero(a > 0)[0]
    if len(nz) == 0:
        return float("inf")
    k = int(nz[0]) - 1
    if k < 0:
        return -1.0
    return (k - 1e-6) / (n - 1)


def upload_lut(lut: np.ndarray):
    return lut_cache.get(np.ascontiguousarray(lut, dtype=np.float32))
