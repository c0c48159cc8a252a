"""Output framebuffer (mirrors `pkg/src/vdikit/image.py:13-22`).

f64 (h, w, 4), premultiplied RGBA, row 0 at the bottom (NDC y = -1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Image:
    data: np.ndarray

    @staticmethod
    def from_array(arr: np.ndarray) -> "Image":
        arr = np.asarray(arr, dtype=np.float64)
        if arr.ndim != 3 or arr.shape[2] != 4:
            raise ValueError(f"expected (h, w, 4), got {arr.shape}")
        return Image(data=arr)

    @property
    def width(self) -> int:
        return self.data.shape[1]

    @property
    def height(self) -> int:
        return self.data.shape[0]

    def __array__(self, dtype=None, copy=None):
        """np.asarray(image): the (h, w, 4) data (the reference's metrics
        accept an Image or an array; metrics.py:25)."""
        return self.data if dtype is None else self.data.astype(dtype, copy=False)

    def rgb(self) -> np.ndarray:
        return np.clip(self.data[..., :3], 0.0, 1.0)
