"""The VDI wire path on the device: VDI1 packing (drop-in for
`vdikit.encode_vdi`, vdi.py:141-159) and LZ4 block compression (drop-in for
`vdikit.lz4.compress`, lz4.py:171-175), plus the fused server path
`compress_vdi` = `lz4.compress(encode_vdi(vdi, grid))` that the reference
server's `generate_fn` / `compress_fn` pair computes (proto.py:283-287,
328-334), with one device->host copy of the compressed block.

The VDI1 bytes are the reference's bit for bit. The LZ4 block is a valid
block of the reference's format that `vdikit.lz4.decompress` (lz4.py:117-168)
inverts exactly; its bytes differ from the reference's serial greedy parse
(the device parses 32 KiB chunks in parallel, csrc/vdi_codec.cu).
"""

from __future__ import annotations

import struct

import numpy as np

from . import _capi
from . import device as dv

MAGIC = b"VDI1"
VERSION = 1
_HEADER = struct.Struct("<4sIIII")   # vdi.py:136
_CAMERA = struct.Struct("<10d")      # vdi.py:137
_AABB = struct.Struct("<6d")         # vdi.py:138
_GRID_DIMS = struct.Struct("<3I")    # vdi.py:139


def vdi1_header(vdi, grid) -> bytes:
    """The first 160 bytes of encode_vdi (vdi.py:143-149)."""
    cam = vdi.gen_camera
    aabb = np.asarray(vdi.volume_aabb, dtype=np.float64).reshape(2, 3)
    return b"".join([
        _HEADER.pack(MAGIC, VERSION, vdi.width, vdi.height, vdi.n_sg),
        _CAMERA.pack(*cam.position, *cam.orientation, cam.fov_y, cam.near, cam.far),
        _AABB.pack(*aabb[0], *aabb[1]),
        _GRID_DIMS.pack(*grid.dims),
    ])


def encode_vdi_device(vdi, grid):
    """Pack on the device. Returns (uint8 device buffer, device u64 length);
    nothing is synchronised."""
    from .raycast import _as_device_grid, _as_device_vdi
    t = dv.require_cuda()
    L = _capi.load()
    vdi = _as_device_vdi(vdi)
    grid = _as_device_grid(grid)
    d = vdi.device()
    gx, gy, gz = grid.dims
    w, h, n = vdi.width, vdi.height, vdi.n_sg
    cap = int(L.vdi_vdi1_max_bytes(w, h, n, gx, gy, gz))
    out = t.empty(cap, dtype=t.uint8, device="cuda")
    out_len = t.zeros(1, dtype=t.int64, device="cuda")
    ws_bytes = int(L.vdi_encode_workspace_bytes(w, h))
    ws = t.empty(ws_bytes, dtype=t.uint8, device="cuda")
    a = _capi.VdiEncodeArgs()
    a.segs, a.counts, a.grid = dv.ptr(d.segs), dv.ptr(d.counts), dv.ptr(grid.device())
    a.out, a.out_len, a.workspace, a.workspace_bytes = (dv.ptr(out), dv.ptr(out_len),
                                                        dv.ptr(ws), ws_bytes)
    hdr = vdi1_header(vdi, grid)
    assert len(hdr) == _capi.VDI1_HEADER_BYTES
    for i, b in enumerate(hdr):
        a.header[i] = b
    a.width, a.height, a.n_sg = w, h, n
    a.gx, a.gy, a.gz = gx, gy, gz
    a.vdi_band_rows, a.vdi_band_world, a.vdi_rows_per_rank = (int(d.band_rows), int(d.world),
                                                              int(d.rows_per_rank))
    _capi.check(L.vdi_encode_vdi1(a, dv.stream_handle()))
    out._keep = ws  # the workspace must outlive the enqueued kernels
    return out, out_len


def encode_vdi(vdi, grid) -> bytes:
    """vdi.py:141-159: the VDI1 byte string (bit-identical to the reference)."""
    out, out_len = encode_vdi_device(vdi, grid)
    n = int(dv.to_host(out_len)[0])
    return dv.to_host(out[:n]).tobytes()


def compress_device(src, n_max: int, n_dev=None, exact: bool = True):
    """LZ4-compress device bytes src[:n] (n = n_dev on the device, else
    n_max). Returns (uint8 device buffer, device u64 length).

    exact=True: the reference's block byte for byte (lz4.py:51-114: one
    serial greedy parse, vdi_lz4_compress_exact). exact=False: the
    chunk-parallel parse (vdi_lz4_compress) -- same format, decoded exactly by
    lz4.decompress, about 2 % larger and much faster."""
    t = dv.require_cuda()
    L = _capi.load()
    dst = t.empty(int(L.vdi_lz4_max_bytes(n_max)), dtype=t.uint8, device="cuda")
    out_len = t.zeros(1, dtype=t.int64, device="cuda")
    ws_fn = L.vdi_lz4_exact_workspace_bytes if exact else L.vdi_lz4_workspace_bytes
    run = L.vdi_lz4_compress_exact if exact else L.vdi_lz4_compress
    ws_bytes = int(ws_fn(n_max))
    ws = t.empty(ws_bytes, dtype=t.uint8, device="cuda")
    _capi.check(run(dv.ptr(src) if n_max else None, int(n_max), dv.ptr(n_dev), dv.ptr(dst),
                    dv.ptr(out_len), dv.ptr(ws), ws_bytes, dv.stream_handle()))
    dst._keep = ws
    return dst, out_len


def compress(data: bytes, exact: bool = True) -> bytes:
    """lz4.py:171-175 compress(): an LZ4 block that lz4.decompress inverts
    (with exact=True, the reference's own bytes)."""
    n = len(data)
    if n == 0:
        return b""
    src = dv.to_device(np.frombuffer(data, dtype=np.uint8))
    dst, out_len = compress_device(src, n, exact=exact)
    m = int(dv.to_host(out_len)[0])
    return dv.to_host(dst[:m]).tobytes()


def compress_vdi(vdi, grid, exact: bool = True):
    """lz4.compress(encode_vdi(vdi, grid)) without the raw bytes leaving the
    device: returns (compressed block, uncompressed length), the two fields
    of the reference's VdiPacket (proto.py:66-86)."""
    raw, raw_len = encode_vdi_device(vdi, grid)
    dst, out_len = compress_device(raw, int(raw.numel()), raw_len, exact=exact)
    lens = dv.to_host(dv.torch().cat([raw_len, out_len]))
    m = int(lens[1])
    return dv.to_host(dst[:m]).tobytes(), int(lens[0])


class BadMagic(ValueError):
    """vdi.py:27-28."""


class VersionMismatch(ValueError):
    """vdi.py:31-32."""


class TruncatedStream(ValueError):
    """vdi.py:35-36."""


def decode_vdi(data: bytes):
    """vdi.py:162-210 decode_vdi: VDI1 bytes -> (Vdi, AccelGrid), device
    resident. The header and the length checks are read on the host (the
    reference's errors: BadMagic, VersionMismatch, TruncatedStream); the
    lists are unpacked on the device (vdi_decode_vdi1_lists) and validated
    there (validate_vdi, InvariantViolation) as the reference does."""
    from .camera import Camera
    from .vdi import AccelGrid, DeviceVdi, InvariantViolation, Vdi, validate_vdi
    t = dv.require_cuda()
    L = _capi.load()
    b = memoryview(data)
    if len(b) < _HEADER.size:
        raise TruncatedStream(f"need {_HEADER.size} bytes, have {len(b)}")
    magic, version, width, height, n_sg = _HEADER.unpack_from(b, 0)
    if magic != MAGIC:
        raise BadMagic(repr(magic))
    if version != VERSION:
        raise VersionMismatch(f"version {version}, expected {VERSION}")
    off = _HEADER.size
    need = off + _CAMERA.size + _AABB.size + _GRID_DIMS.size
    if len(b) < need:
        raise TruncatedStream(f"need {need} bytes, have {len(b)}")
    camvals = _CAMERA.unpack_from(b, off)
    off += _CAMERA.size
    aabbvals = _AABB.unpack_from(b, off)
    off += _AABB.size
    gdims = _GRID_DIMS.unpack_from(b, off)
    off += _GRID_DIMS.size
    n = width * height
    if len(b) < off + 2 * n:
        raise TruncatedStream(f"need {off + 2 * n} bytes, have {len(b)}")
    counts_u16 = np.frombuffer(b, "<u2", n, off)
    total = int(counts_u16.sum(dtype=np.int64))  # sizes the stream (vdi.py:182-183)
    ng = gdims[0] * gdims[1] * gdims[2]
    end = off + 2 * n + 24 * total + 4 * ng
    if len(b) < end:
        raise TruncatedStream(f"need {end} bytes, have {len(b)}")
    if len(b) > end:
        raise TruncatedStream(f"{len(b) - end} trailing bytes")
    over = np.flatnonzero(counts_u16 > n_sg)
    if over.size:  # vdi.py:199-201: the first such list in row-major order
        ly, lx = divmod(int(over[0]), width)
        raise InvariantViolation(f"list ({lx},{ly}) count {int(counts_u16[over[0]])} "
                                 f"> n_sg {n_sg}")
    cam = Camera(position=camvals[0:3], orientation=camvals[3:7], fov_y=camvals[7],
                 near=camvals[8], far=camvals[9], viewport=(width, height))
    aabb = np.array(aabbvals, dtype=np.float64).reshape(2, 3)
    src = dv.to_device(np.frombuffer(b, np.uint8, end - 4 * ng, 0))
    counts = t.empty((height, width), dtype=t.int32, device="cuda")
    segs = t.empty((max(n, 1), (6 * n_sg + 3) & ~3), dtype=t.float32, device="cuda")
    ws = t.empty(int(L.vdi_encode_workspace_bytes(width, height)), dtype=t.uint8, device="cuda")
    _capi.check(L.vdi_decode_vdi1_lists(dv.ptr(src), width, height, n_sg, dv.ptr(counts),
                                        dv.ptr(segs), dv.ptr(ws), int(ws.numel()),
                                        dv.stream_handle()))
    grid = np.frombuffer(b, "<u4", ng, end - 4 * ng).reshape(gdims[2], gdims[1], gdims[0]).copy()
    vdi = Vdi(width, height, n_sg, None, None, cam, aabb,
              _device=DeviceVdi(counts=counts, segs=segs))
    agrid = AccelGrid(tuple(gdims), grid, cam.near, cam.far)
    validate_vdi(vdi)
    return vdi, agrid
