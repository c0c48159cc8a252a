"""ctypes binding of libvdi_b200.so (include/vdi_b200.h).

The structures below mirror the header field for field. Loading fails loudly:
there is no CPU fallback for the product path.
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libvdi_b200.so")

VOXEL = {"u8": 0, "u16": 1, "f32": 2}
VOXEL_CELLS = 16  # flag: VdiGenArgs.volume holds vdi_volume_cells() records
_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int32


class VdiGenArgs(ctypes.Structure):
    _fields_ = [
        ("volume", _P), ("lut", _P), ("brick_max", _P), ("counts", _P), ("segs", _P), ("gammas", _P),
        ("passes", _P), ("samples", _P), ("workspace", _P), ("workspace_bytes", ctypes.c_size_t),
        ("pv", _D * 16), ("inv_pv", _D * 16), ("eye", _D * 3), ("aabb", _D * 6),
        ("eps", _D), ("gamma_init", _D), ("step", _D), ("lref", _D), ("ess_max", _D),
        ("voxel_type", _I), ("nx", _I), ("ny", _I), ("nz", _I), ("lut_n", _I),
        ("width", _I), ("height", _I), ("n_sg", _I), ("delta", _I),
        ("band_rows", _I), ("band_stride", _I), ("band_offset", _I), ("brick_log2", _I),
        ("sub_origin", _I * 3), ("sub_dims", _I * 3), ("sub_oob", _P),
        ("row_base", _I), ("row_count", _I),
    ]


class VdiGridArgs(ctypes.Structure):
    _fields_ = [
        ("segs", _P), ("counts", _P), ("grid", _P),
        ("near", _D), ("far", _D), ("proj_a", _D), ("proj_b", _D),
        ("width", _I), ("height", _I), ("n_sg", _I), ("gx", _I), ("gy", _I), ("gz", _I),
        ("band_rows", _I), ("band_stride", _I), ("band_offset", _I), ("clear", _I),
        ("row_base", _I), ("row_count", _I),
    ]


class VdiRenderArgs(ctypes.Structure):
    _fields_ = [
        ("segs", _P), ("counts", _P), ("grid", _P), ("image", _P),
        ("lists_visited", _P), ("segs_intersected", _P), ("lists_searched", _P),
        ("stat_sums", _P),
        ("gen_pv", _D * 16), ("gen_inv_pv", _D * 16), ("new_inv_pv", _D * 16),
        ("eye", _D * 3), ("aabb", _D * 6), ("bg", _D * 4),
        ("near", _D), ("far", _D), ("proj_a", _D), ("proj_b", _D), ("early_term", _D),
        ("vdi_w", _I), ("vdi_h", _I), ("n_sg", _I), ("gx", _I), ("gy", _I), ("gz", _I),
        ("out_w", _I), ("out_h", _I), ("use_ess", _I),
        ("vdi_band_rows", _I), ("vdi_band_world", _I), ("vdi_rows_per_rank", _I),
        ("band_rows", _I), ("band_stride", _I), ("band_offset", _I),
        ("list_tiles", _P), ("grid_zmask", _P), ("lists_sorted", _I), ("counters_exact", _I),
        ("vdi_row_map", _P), ("list_range", _P), ("tile_counter", _P),
    ]


class VdiDvrArgs(ctypes.Structure):
    _fields_ = [
        ("volume", _P), ("lut", _P), ("brick_max", _P), ("image", _P), ("samples", _P),
        ("stat_sums", _P), ("workspace", _P),
        ("pv", _D * 16), ("inv_pv", _D * 16), ("eye", _D * 3), ("aabb", _D * 6), ("bg", _D * 4),
        ("step", _D), ("lref", _D), ("early_term", _D), ("ess_max", _D),
        ("voxel_type", _I), ("nx", _I), ("ny", _I), ("nz", _I), ("lut_n", _I),
        ("width", _I), ("height", _I), ("band_rows", _I), ("band_stride", _I),
        ("band_offset", _I), ("brick_log2", _I),
    ]


DVR_WORKSPACE_BYTES = 256


class VdiPreviewArgs(ctypes.Structure):
    _fields_ = [
        ("segs", _P), ("counts", _P), ("grid", _P), ("image", _P), ("cell_samples", _P),
        ("stat_sums", _P), ("workspace", _P),
        ("gen_pv", _D * 16), ("gen_inv_pv", _D * 16), ("new_inv_pv", _D * 16),
        ("eye", _D * 3), ("aabb", _D * 6), ("bg", _D * 4),
        ("near", _D), ("far", _D), ("proj_a", _D), ("proj_b", _D), ("d_r", _D),
        ("early_term", _D),
        ("vdi_w", _I), ("vdi_h", _I), ("n_sg", _I), ("gx", _I), ("gy", _I), ("gz", _I),
        ("out_w", _I), ("out_h", _I),
        ("vdi_band_rows", _I), ("vdi_band_world", _I), ("vdi_rows_per_rank", _I),
    ]


PREVIEW_WORKSPACE_BYTES = 256
VDI1_HEADER_BYTES = 160


class VdiEncodeArgs(ctypes.Structure):
    _fields_ = [
        ("segs", _P), ("counts", _P), ("grid", _P), ("out", _P), ("out_len", _P),
        ("workspace", _P), ("workspace_bytes", ctypes.c_size_t),
        ("header", ctypes.c_uint8 * VDI1_HEADER_BYTES),
        ("width", _I), ("height", _I), ("n_sg", _I), ("gx", _I), ("gy", _I), ("gz", _I),
        ("vdi_band_rows", _I), ("vdi_band_world", _I), ("vdi_rows_per_rank", _I),
    ]


class VdiValidateArgs(ctypes.Structure):
    _fields_ = [
        ("segs", _P), ("counts", _P), ("result", _P),
        ("width", _I), ("height", _I), ("n_sg", _I),
        ("vdi_band_rows", _I), ("vdi_band_world", _I), ("vdi_rows_per_rank", _I),
    ]

EXPORTS = ["vdi_last_error", "vdi_abi_version", "vdi_gen_workspace_bytes",
           "vdi_gen_workspace_min_bytes", "vdi_gen_launch",
           "vdi_grid_launch", "vdi_render_launch", "vdi_dvr_launch",
           "vdi_preview_launch", "vdi_bilinear_upsample", "vdi_vdi1_max_bytes",
           "vdi_encode_workspace_bytes", "vdi_encode_vdi1", "vdi_lz4_max_bytes",
           "vdi_lz4_workspace_bytes", "vdi_lz4_compress",
           "vdi_lz4_exact_workspace_bytes", "vdi_lz4_compress_exact", "vdi_validate", "vdi_synth_rm_u8",
           "vdi_gen_rays", "vdi_composite_lists", "vdi_dda_cells", "vdi_project_rays",
           "vdi_decode_vdi1_lists", "vdi_find_first_batch",
           "vdi_volume_brick_max", "vdi_selftest_arith", "vdi_segs_to_aos",
           "vdi_segs_from_aos", "vdi_volume_cells_bytes", "vdi_volume_cells", "vdi_volume_cells_masked",
           "vdi_list_tiles_words", "vdi_list_tiles", "vdi_grid_zmask", "vdi_list_ranges"]

_lib = None


class VdiError(RuntimeError):
    pass


def load():
    """Load the built library (never builds, never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise VdiError(f"{LIB_PATH} is not built; run `python -m paper_2206_08660_b200.build` "
                       "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.vdi_last_error.restype = ctypes.c_char_p
    L.vdi_abi_version.restype = ctypes.c_int
    L.vdi_gen_workspace_bytes.restype = ctypes.c_size_t
    L.vdi_gen_workspace_bytes.argtypes = [ctypes.POINTER(VdiGenArgs)]
    L.vdi_gen_workspace_min_bytes.restype = ctypes.c_size_t
    L.vdi_gen_workspace_min_bytes.argtypes = [ctypes.POINTER(VdiGenArgs)]
    L.vdi_gen_launch.argtypes = [ctypes.POINTER(VdiGenArgs), _P]
    L.vdi_grid_launch.argtypes = [ctypes.POINTER(VdiGridArgs), _P]
    L.vdi_render_launch.argtypes = [ctypes.POINTER(VdiRenderArgs), _P]
    L.vdi_dvr_launch.argtypes = [ctypes.POINTER(VdiDvrArgs), _P]
    L.vdi_preview_launch.argtypes = [ctypes.POINTER(VdiPreviewArgs), _P]
    L.vdi_vdi1_max_bytes.argtypes = [_I, _I, _I, _I, _I, _I]
    L.vdi_vdi1_max_bytes.restype = ctypes.c_size_t
    L.vdi_encode_workspace_bytes.argtypes = [_I, _I]
    L.vdi_encode_workspace_bytes.restype = ctypes.c_size_t
    L.vdi_encode_vdi1.argtypes = [ctypes.POINTER(VdiEncodeArgs), _P]
    L.vdi_lz4_max_bytes.argtypes = [ctypes.c_size_t]
    L.vdi_lz4_max_bytes.restype = ctypes.c_size_t
    L.vdi_lz4_workspace_bytes.argtypes = [ctypes.c_size_t]
    L.vdi_lz4_workspace_bytes.restype = ctypes.c_size_t
    L.vdi_lz4_compress.argtypes = [_P, ctypes.c_size_t, _P, _P, _P, _P, ctypes.c_size_t, _P]
    L.vdi_lz4_exact_workspace_bytes.argtypes = [ctypes.c_size_t]
    L.vdi_lz4_exact_workspace_bytes.restype = ctypes.c_size_t
    L.vdi_lz4_compress_exact.argtypes = [_P, ctypes.c_size_t, _P, _P, _P, _P, ctypes.c_size_t, _P]
    L.vdi_validate.argtypes = [ctypes.POINTER(VdiValidateArgs), _P]
    L.vdi_decode_vdi1_lists.argtypes = [_P, _I, _I, _I, _P, _P, _P, ctypes.c_size_t, _P]
    L.vdi_gen_rays.argtypes = [ctypes.POINTER(VdiGenArgs), _P, _P, ctypes.c_int64, _I, _P]
    L.vdi_composite_lists.argtypes = [_P, _P, _I, _I, _I, _D, _P, _P, _P]
    L.vdi_dda_cells.argtypes = [_P, ctypes.c_int64, _I, _I, _I, _P, _P, _P, _P]
    L.vdi_project_rays.argtypes = [_P, ctypes.c_int64, _P, _P, _P, _P, _P]
    L.vdi_synth_rm_u8.argtypes = [_P, _I, _I, _I, _P, _P, ctypes.c_float, ctypes.c_uint32, _P]
    L.vdi_bilinear_upsample.argtypes = [_P, _I, _I, _P, _I, _I, _I, _P]
    L.vdi_find_first_batch.argtypes = [_P, _P, _P, _I, _P, _P, _P, _P, _P, ctypes.c_int64, _P]
    L.vdi_volume_brick_max.argtypes = [_P, _I, _I, _I, _I, _I, _P, _P]
    L.vdi_volume_brick_max.restype = ctypes.c_int
    L.vdi_volume_cells_bytes.argtypes = [_I, _I, _I, _I]
    L.vdi_volume_cells_bytes.restype = ctypes.c_size_t
    L.vdi_volume_cells.argtypes = [_P, _I, _I, _I, _I, _P, _P]
    L.vdi_volume_cells.restype = ctypes.c_int
    L.vdi_volume_cells_masked.argtypes = [_P, _I, _I, _I, _I, _P, _I, _D, _P, _P]
    L.vdi_volume_cells_masked.restype = ctypes.c_int
    L.vdi_selftest_arith.argtypes = [ctypes.c_int64, ctypes.c_uint64, _P, _P]
    L.vdi_selftest_arith.restype = ctypes.c_int
    L.vdi_list_tiles.argtypes = [ctypes.POINTER(VdiRenderArgs), _P, _P]
    L.vdi_list_tiles_words.argtypes = [_I, _I]
    L.vdi_list_tiles_words.restype = ctypes.c_size_t
    L.vdi_grid_zmask.argtypes = [_P, _I, _I, _I, _P, _P]
    L.vdi_list_ranges.argtypes = [_P, _P, ctypes.c_int64, _I, _P, _P]
    L.vdi_segs_to_aos.argtypes = [_P, _P, ctypes.c_int64, _I, _P]
    L.vdi_segs_from_aos.argtypes = [_P, _P, ctypes.c_int64, _I, _P]
    for name in ("vdi_gen_launch", "vdi_grid_launch", "vdi_render_launch", "vdi_dvr_launch",
                 "vdi_preview_launch", "vdi_bilinear_upsample", "vdi_encode_vdi1",
                 "vdi_decode_vdi1_lists", "vdi_lz4_compress", "vdi_lz4_compress_exact",
                 "vdi_validate", "vdi_synth_rm_u8",
                 "vdi_gen_rays", "vdi_composite_lists", "vdi_dda_cells", "vdi_project_rays",
                 "vdi_find_first_batch", "vdi_segs_to_aos", "vdi_segs_from_aos",
                 "vdi_list_tiles", "vdi_grid_zmask", "vdi_list_ranges"):
        getattr(L, name).restype = ctypes.c_int
    if L.vdi_abi_version() != 8:
        raise VdiError("libvdi_b200.so ABI mismatch")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        raise VdiError(f"vdi_b200 error {rc}: {load().vdi_last_error().decode()}")


def fill(arr, values) -> None:
    for i, v in enumerate(values):
        arr[i] = float(v)
