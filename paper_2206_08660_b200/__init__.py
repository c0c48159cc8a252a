"""B200-native VDI generation and VDI raycasting (arXiv 2206.08660).

Drop-in for the hot path of the reference package `vdikit`
(/root/reference/pkg/src/vdikit): `generate_vdi` (generate.py:444-479) and
`render_vdi` (raycast.py:459-491) keep the reference's signatures and return
types, and run on hand-written sm_100a CUDA kernels behind the C ABI in
include/vdi_b200.h. There is no CPU fallback: without the built extension
and a CUDA device the compute entry points raise.
"""

from .camera import Camera, Ray, generate_ray, look_at, orbit_camera
from .image import Image
from .volume import TransferFunction, Volume, grayscale_tf, make_volume

__version__ = "0.1.0"

_LAZY = {
    "GenParams": "generate", "GenStats": "generate", "generate_vdi": "generate",
    "RenderOptions": "raycast", "RenderStats": "raycast", "render_vdi": "raycast",
    "find_first_supersegment": "raycast", "composite_lists": "raycast",
    "dda_traverse": "raycast", "project_ray_to_ndc": "raycast", "opacity_correct": "raycast",
    "terminate_check": "generate", "generate_list": "generate", "find_gamma": "generate",
    "Vdi": "vdi", "AccelGrid": "vdi", "default_grid_dims": "vdi",
    "validate_vdi": "vdi",
    "FrameStream": "stream", "FrameResult": "stream",
    "render_dvr": "dvr",
    "render_preview": "preview", "PreviewParams": "preview", "PreviewStats": "preview",
    "PiController": "preview", "pi_update": "preview", "samples_in_cell": "preview",
    "bilinear_upsample": "preview",
    "encode_vdi": "codec", "compress": "codec", "compress_vdi": "codec",
    "decode_vdi": "codec",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = ["Camera", "Ray", "generate_ray", "look_at", "orbit_camera", "Image",
           "TransferFunction", "Volume", "grayscale_tf", "make_volume",
           *_LAZY]
