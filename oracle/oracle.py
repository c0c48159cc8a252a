"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

The oracle restates the reference's numba kernels in C (vdi_oracle.c, which
cites generate.py / raycast.py line by line). Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline leg import this module; the product package never
does. Array conventions are the reference's: segs (H, W, n_sg, 6) f32 AoS,
image (h, w, 4) f64, grid (gz, gy, gx) u32.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libvdi_oracle.so")
_lib = None

_f32 = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64 = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u32 = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_vp = ctypes.c_void_p
_int = ctypes.c_int
_dbl = ctypes.c_double


def build(force: bool = False) -> str:
    """Compile libvdi_oracle.so with the committed Makefile."""
    src = os.path.join(_HERE, "vdi_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.vdio_generate.argtypes = [
            _f32, _int, _int, _int, _f32, _int, _f64, _f64, _f64, _f64,
            _int, _int, _int, _int, _dbl, _dbl, _dbl, _dbl,
            _vp, _int, _int, _i32, _f32, _f64, _i32, _i64]
        _u8v = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        L.vdio_generate_u8.argtypes = [_u8v] + L.vdio_generate.argtypes[1:]
        L.vdio_accumulate_grid.argtypes = [
            _i32, _f32, _int, _int, _int, _int, _int, _int,
            _dbl, _dbl, _dbl, _dbl, _u32]
        L.vdio_render.argtypes = [
            _f32, _i32, _int, _int, _int, _f64, _f64, _f64, _f64, _f64,
            _int, _int, _int, _u32, _int, _int, _int,
            _dbl, _dbl, _dbl, _dbl, _dbl, _f64,
            _vp, _int, _int, _f64, _i64, _i64, _i64]
        L.vdio_find_first.argtypes = [_f32, _f32, ctypes.c_int64, _dbl, _dbl,
                                      ctypes.c_int64,
                                      ctypes.POINTER(ctypes.c_int64)]
        L.vdio_find_first.restype = ctypes.c_int64
        L.vdio_dvr.argtypes = [
            _f32, _int, _int, _int, _f32, _int, _f64, _f64, _f64, _f64,
            _int, _int, _dbl, _dbl, _dbl, _f64, _vp, _int, _int, _f64, _vp]
        L.vdio_preview.argtypes = [
            _f32, _i32, _int, _int, _int, _f64, _f64, _f64, _f64, _f64,
            _int, _int, _u32, _int, _int, _int, _dbl, _dbl, _dbl, _dbl,
            _dbl, _dbl, _f64, _int, _f64, _i64]
        L.vdio_preview.restype = ctypes.c_int64
        _u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        L.vdio_lz4_compress.argtypes = [_u8, ctypes.c_int64, _u8]
        L.vdio_lz4_compress.restype = ctypes.c_int64
        L.vdio_lz4_decompress.argtypes = [_u8, ctypes.c_int64, _u8, ctypes.c_int64]
        L.vdio_lz4_decompress.restype = ctypes.c_int64
        L.vdio_max_threads.restype = _int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().vdio_max_threads())


def _m(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))


def _rows(rows):
    if rows is None:
        return None, 0, None
    r = np.ascontiguousarray(rows, dtype=np.int32)
    return r.ctypes.data_as(ctypes.c_void_p), len(r), r


def generate(vol_norm, lut, pv, inv_pv, eye, aabb, width, height, n_sg, delta,
             eps, gamma_init, step, lref, rows=None, threads=0, compact=False):
    """_generate_kernel (generate.py:276-319) + executed-sample counter.

    vol_norm is the f32 (nz, ny, nx) array R samples (Volume.normalized), or
    the raw u8 voxels it is derived from (normalised identically on the fly)."""
    u8 = isinstance(vol_norm, np.ndarray) and vol_norm.dtype == np.uint8
    vol = np.ascontiguousarray(vol_norm) if u8 else np.ascontiguousarray(vol_norm, np.float32)
    nz, ny, nx = vol.shape
    lut = np.ascontiguousarray(lut, dtype=np.float32)
    oh = len(rows) if (compact and rows is not None) else height
    counts = np.zeros((oh, width), np.int32)
    segs = np.zeros((oh, width, n_sg, 6), np.float32)
    gammas = np.zeros((oh, width), np.float64)
    passes = np.zeros((oh, width), np.int32)
    samples = np.zeros((oh, width), np.int64)
    rp, nr, _keep = _rows(rows)
    if compact and rows is not None:
        nr = -nr
    fn = lib().vdio_generate_u8 if u8 else lib().vdio_generate
    fn(vol, nx, ny, nz, lut, lut.shape[0], _m(pv), _m(inv_pv),
                        _m(eye), _m(aabb), width, height, n_sg, delta,
                        float(eps), float(gamma_init), float(step), float(lref),
                        rp, nr, threads, counts, segs, gammas, passes, samples)
    return dict(counts=counts, segs=segs, gammas=gammas, passes=passes,
                samples=samples)  # compact: rows in the order given


def accumulate_grid(counts, segs, dims, near, far, proj_a, proj_b):
    """_accumulate_grid (generate.py:322-346)."""
    gx, gy, gz = dims
    height, width, n_sg, _ = segs.shape
    g = np.zeros((gz, gy, gx), np.uint32)
    lib().vdio_accumulate_grid(np.ascontiguousarray(counts, np.int32),
                               np.ascontiguousarray(segs, np.float32),
                               width, height, n_sg, gx, gy, gz, float(near),
                               float(far), float(proj_a), float(proj_b), g)
    return g


def depth_consts(near, far):
    """generate.py:349-354 / raycast.py:471-472."""
    return (far + near) / (far - near), 2.0 * far * near / (far - near)


def render(segs, counts, gen_pv, gen_inv_pv, aabb, new_inv_pv, eye, out_w,
           out_h, grid, near, far, use_ess=True, early_term=0.999,
           bg=(0.0, 0.0, 0.0, 1.0), rows=None, threads=0):
    """_render_kernel (raycast.py:275-456) with per-pixel counters."""
    segs = np.ascontiguousarray(segs, np.float32)
    vdi_h, vdi_w, n_sg, _ = segs.shape
    grid = np.ascontiguousarray(grid, np.uint32)
    gz, gy, gx = grid.shape
    pa, pb = depth_consts(near, far)
    img = np.zeros((out_h, out_w, 4), np.float64)
    lv = np.zeros((out_h, out_w), np.int64)
    si = np.zeros((out_h, out_w), np.int64)
    ls = np.zeros((out_h, out_w), np.int64)
    rp, nr, _keep = _rows(rows)
    lib().vdio_render(segs, np.ascontiguousarray(counts, np.int32), vdi_w,
                      vdi_h, n_sg, _m(gen_pv), _m(gen_inv_pv), _m(aabb),
                      _m(new_inv_pv), _m(eye), out_w, out_h, int(bool(use_ess)),
                      grid, gx, gy, gz, float(near), float(far), pa, pb,
                      float(early_term), _m(bg), rp, nr, threads, img, lv, si, ls)
    return dict(image=img, lists_visited=lv, segs_intersected=si,
                lists_searched=ls)


def find_first(fronts, backs, count, d_entry, d_exit, p):
    """_find_first (raycast.py:79-141): returns (index or -1, seed)."""
    fr = np.ascontiguousarray(fronts, np.float32)
    bk = np.ascontiguousarray(backs, np.float32)
    seed = ctypes.c_int64(0)
    idx = lib().vdio_find_first(fr, bk, int(count), float(d_entry),
                                float(d_exit), int(p), ctypes.byref(seed))
    return int(idx), int(seed.value)


def dvr(vol_norm, lut, pv, inv_pv, eye, aabb, width, height, step, lref,
        early_term=0.999, bg=(0.0, 0.0, 0.0, 1.0), rows=None, threads=0,
        with_samples=False):
    """_dvr_kernel (dvr.py:21-89): image (h, w, 4) f64 [, executed samples]."""
    vol = np.ascontiguousarray(vol_norm, dtype=np.float32)
    nz, ny, nx = vol.shape
    lut = np.ascontiguousarray(lut, dtype=np.float32)
    img = np.zeros((height, width, 4), np.float64)
    smp = np.zeros((height, width), np.int64) if with_samples else None
    rp, nr, _keep = _rows(rows)
    lib().vdio_dvr(vol, nx, ny, nz, lut, lut.shape[0], _m(pv), _m(inv_pv), _m(eye),
                   _m(aabb), width, height, float(step), float(lref), float(early_term),
                   _m(bg), rp, nr, threads, img,
                   None if smp is None else smp.ctypes.data_as(ctypes.c_void_p))
    return (img, smp) if with_samples else img


def preview_lowres(segs, counts, gen_pv, gen_inv_pv, aabb, new_inv_pv, eye, out_w, out_h,
                   grid, near, far, d_r, early_term=0.999, bg=(0.0, 0.0, 0.0, 1.0),
                   threads=0):
    """_preview_kernel (preview.py:49-205): low-res image, total samples,
    per-cell samples (gz, gy, gx) i64."""
    segs = np.ascontiguousarray(segs, np.float32)
    vdi_h, vdi_w, n_sg, _ = segs.shape
    grid = np.ascontiguousarray(grid, np.uint32)
    gz, gy, gx = grid.shape
    pa, pb = depth_consts(near, far)
    img = np.zeros((out_h, out_w, 4), np.float64)
    cells = np.zeros((gz, gy, gx), np.int64)
    total = lib().vdio_preview(segs, np.ascontiguousarray(counts, np.int32), vdi_w, vdi_h,
                               n_sg, _m(gen_pv), _m(gen_inv_pv), _m(aabb), _m(new_inv_pv),
                               _m(eye), out_w, out_h, grid, gx, gy, gz, float(near),
                               float(far), pa, pb, float(d_r), float(early_term), _m(bg),
                               threads, img, cells)
    return img, int(total), cells


def bilinear_upsample(arr, out_w, out_h):
    """preview.py:208-223, restated with the same numpy expressions."""
    h, w = arr.shape[:2]
    if (w, h) == (out_w, out_h):
        return arr
    xs = (np.arange(out_w) + 0.5) * w / out_w - 0.5
    ys = (np.arange(out_h) + 0.5) * h / out_h - 0.5
    x0 = np.clip(np.floor(xs).astype(np.int64), 0, w - 1)
    y0 = np.clip(np.floor(ys).astype(np.int64), 0, h - 1)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    fx = np.clip(xs - x0, 0.0, 1.0)[None, :, None]
    fy = np.clip(ys - y0, 0.0, 1.0)[:, None, None]
    top = arr[y0[:, None], x0[None, :]] * (1 - fx) + arr[y0[:, None], x1[None, :]] * fx
    bot = arr[y1[:, None], x0[None, :]] * (1 - fx) + arr[y1[:, None], x1[None, :]] * fx
    return top * (1 - fy) + bot * fy


def lz4_compress(data: bytes) -> bytes:
    """lz4.py:51-114 + 171-175 compress()."""
    src = np.frombuffer(data, dtype=np.uint8).copy()
    dst = np.empty(len(data) + len(data) // 255 + 16, dtype=np.uint8)
    n = lib().vdio_lz4_compress(src, len(src), dst)
    return dst[:n].tobytes()


def lz4_decompress(data: bytes, uncompressed_len: int) -> bytes:
    """lz4.py:117-168 + 178-189 decompress(); raises ValueError like
    DecompressFailure."""
    if uncompressed_len == 0:
        if len(data) != 0 and data != b"\x00":
            raise ValueError("nonempty block for empty payload")
        return b""
    src = np.frombuffer(data, dtype=np.uint8).copy()
    dst = np.empty(uncompressed_len, dtype=np.uint8)
    n = lib().vdio_lz4_decompress(src, len(src), dst, uncompressed_len)
    if n != uncompressed_len:
        raise ValueError(f"decoded {n} bytes, expected {uncompressed_len}")
    return dst.tobytes()


def encode_vdi(width, height, n_sg, counts, segs, cam_vals, aabb, grid):
    """vdi.py:141-159 encode_vdi: the VDI1 little-endian byte layout.
    cam_vals = (pos3, quat4, fov_y, near, far); segs (H, W, n_sg, 6) AoS;
    grid (gz, gy, gx)."""
    import struct
    gz, gy, gx = grid.shape
    parts = [struct.pack("<4sIIII", b"VDI1", 1, width, height, n_sg),
             struct.pack("<10d", *cam_vals),
             struct.pack("<6d", *np.asarray(aabb, np.float64).reshape(6)),
             struct.pack("<3I", gx, gy, gz),
             np.asarray(counts).astype("<u2").tobytes()]
    mask = np.arange(n_sg)[None, None, :] < np.asarray(counts)[:, :, None]
    parts.append(np.asarray(segs, np.float32)[mask].astype("<f4").tobytes())
    parts.append(np.asarray(grid).astype("<u4").tobytes())
    return b"".join(parts)
