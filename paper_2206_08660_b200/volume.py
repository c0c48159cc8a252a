"""Volumes and transfer functions (host side).

Mirrors `pkg/src/vdikit/volume.py`:
  * `Volume` (volume.py:30-60): scalar brick `data` in (nz, ny, nx) x-fastest
    order, per-axis spacing, AABB = [0, dims * spacing]; `normalized` is the
    f32 copy every reference kernel samples.
  * `TransferFunction` (volume.py:125-147): control points baked into a
    256 x 4 f32 LUT with np.interp, clipped to [0, 1].

B200 difference: the device never needs the 4 B/voxel f32 copy for integer
volumes. `float(v) / 255.0f` rounds identically to numpy's
`data.astype(f32) / 255` (IEEE division), so u8/u16 volumes are uploaded raw
(1-2 B/voxel) and normalised inside the sampler. `voxel_type="f32"` is the
B200-side extension for float volumes (BASELINE configs 1, 2, 4); the
reference reaches the same state with `Volume(..., normalized=arr)`
(volume.py:48).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

VOXEL_DTYPES = {"u8": np.uint8, "u16": np.uint16, "f32": np.float32}
VOXEL_MAX = {"u8": 255.0, "u16": 65535.0, "f32": 1.0}


class SizeMismatch(ValueError):
    pass


class UnsupportedVoxelType(ValueError):
    pass


@dataclass(frozen=True)
class Volume:
    dims: tuple                 # (nx, ny, nz)
    voxel_type: str             # "u8" | "u16" | "f32"
    spacing: tuple
    data: np.ndarray            # (nz, ny, nx)
    value_range: tuple
    normalized: np.ndarray = field(repr=False, default=None)

    def __post_init__(self):
        nx, ny, nz = self.dims
        if min(self.dims) < 2:
            raise ValueError("dims components must be >= 2 for trilinear sampling")
        if min(self.spacing) <= 0:
            raise ValueError("spacing components must be > 0")
        if self.data.size != nx * ny * nz:
            raise SizeMismatch(f"data has {self.data.size} voxels, dims say {nx*ny*nz}")
        if self.voxel_type not in VOXEL_DTYPES:
            raise UnsupportedVoxelType(self.voxel_type)
        # `normalized` is materialised lazily: the device path uploads the raw
        # brick, so building a 4 B/voxel host copy of a 3 GiB volume up front
        # would only cost host RAM.
        object.__setattr__(self, "_norm_derived",
                           object.__getattribute__(self, "normalized") is None)

    def __getattribute__(self, name):
        if name == "normalized":
            v = object.__getattribute__(self, "normalized")
            if v is None:
                data = object.__getattribute__(self, "data")
                vt = object.__getattribute__(self, "voxel_type")
                if vt == "f32":
                    v = np.ascontiguousarray(data, dtype=np.float32)
                else:
                    v = data.astype(np.float32) / np.float32(VOXEL_MAX[vt])
                object.__setattr__(self, "normalized", v)
            return v
        return object.__getattribute__(self, name)

    @property
    def normalized_is_derived(self) -> bool:
        """True when sampling may use `data` and normalise on the fly."""
        return object.__getattribute__(self, "_norm_derived")

    @property
    def world_size(self) -> np.ndarray:
        return np.array(self.dims, dtype=np.float64) * np.array(self.spacing)

    @property
    def aabb(self) -> np.ndarray:
        return np.stack([np.zeros(3), self.world_size])


class DeviceVolume:
    """A volume that lives only in device memory (a torch tensor (nz, ny, nx)
    of the voxel type), e.g. one synthesised on the GPU. It carries the
    Volume attributes the path reads (dims, voxel_type, spacing, aabb,
    world_size); `data` / `normalized` copy it to the host on first use (for
    checkers only -- the device path never needs them)."""

    normalized_is_derived = True

    def __init__(self, device_data, voxel_type: str, spacing=(1.0, 1.0, 1.0), full_dims=None,
                 origin=(0, 0, 0)):
        """full_dims / origin: device_data is only the resident box
        [origin, origin + shape) of a full_dims volume (one rank's bricks)."""
        if voxel_type not in VOXEL_DTYPES:
            raise UnsupportedVoxelType(voxel_type)
        nz, ny, nx = (int(v) for v in device_data.shape)
        if min(nx, ny, nz) < 2:
            raise ValueError("dims components must be >= 2 for trilinear sampling")
        self.device_data = device_data
        self.box_dims = (nx, ny, nz)
        self.origin = tuple(int(v) for v in origin)
        self.dims = tuple(int(v) for v in full_dims) if full_dims is not None else (nx, ny, nz)
        self.is_sub = full_dims is not None
        self.voxel_type = voxel_type
        self.spacing = tuple(float(v) for v in spacing)
        self._host = None

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            self._host = self.device_data.cpu().numpy()
        return self._host

    @property
    def normalized(self) -> np.ndarray:
        d = self.data
        if self.voxel_type == "f32":
            return d
        return d.astype(np.float32) / np.float32(VOXEL_MAX[self.voxel_type])

    @property
    def value_range(self) -> tuple:
        return (float(self.device_data.min()), float(self.device_data.max()))

    @property
    def world_size(self) -> np.ndarray:
        return np.array(self.dims, dtype=np.float64) * np.array(self.spacing)

    @property
    def aabb(self) -> np.ndarray:
        return np.stack([np.zeros(3), self.world_size])


def make_volume(data: np.ndarray, voxel_type: str, spacing=(1.0, 1.0, 1.0)) -> Volume:
    """Wrap a (nz, ny, nx) scalar array (volume.py:63-75)."""
    if voxel_type not in VOXEL_DTYPES:
        raise UnsupportedVoxelType(voxel_type)
    data = np.ascontiguousarray(data, dtype=VOXEL_DTYPES[voxel_type])
    nz, ny, nx = data.shape
    return Volume(dims=(nx, ny, nz), voxel_type=voxel_type,
                  spacing=tuple(float(s) for s in spacing), data=data,
                  value_range=(float(data.min()), float(data.max())))


@dataclass(frozen=True)
class TransferFunction:
    """Piecewise-linear RGBA over normalised scalar, baked to a LUT."""

    control_points: tuple
    resolution: int = 256
    lut: np.ndarray = field(repr=False, default=None)

    def __post_init__(self):
        pts = [tuple(float(v) for v in p) for p in self.control_points]
        s = [p[0] for p in pts]
        if s[0] != 0.0 or s[-1] != 1.0:
            raise ValueError("first control point must be at 0, last at 1")
        if any(b <= a for a, b in zip(s, s[1:])):
            raise ValueError("control points must be strictly ascending in scalar")
        object.__setattr__(self, "control_points", tuple(pts))
        if self.lut is None:
            xs = np.linspace(0.0, 1.0, self.resolution)
            arr = np.array(pts)
            chans = [np.interp(xs, arr[:, 0], arr[:, 1 + c]) for c in range(4)]
            lut = np.stack(chans, axis=1).astype(np.float32)
            object.__setattr__(self, "lut", np.clip(lut, 0.0, 1.0))


def grayscale_tf(alpha: float = 1.0) -> TransferFunction:
    return TransferFunction(((0.0, 0, 0, 0, 0.0), (1.0, 1, 1, 1, alpha)))
