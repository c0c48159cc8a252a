"""The device wire path (vdi_encode_vdi1, vdi_lz4_compress) and the device
validator (vdi_validate) vs the reference.

- encode_vdi: the VDI1 bytes equal the reference's (sha256 from codec.npz,
  made by vdikit.encode_vdi) and the oracle's, for every committed VDI.
- LZ4, exact mode (the default; vdi_lz4_compress_exact): the block equals
  the reference's byte for byte -- its own blocks in codec.npz (made by
  vdikit.lz4.compress) and, for generated inputs (chunk-boundary sizes,
  unaligned sources, full C1 / C3 VDIs), the pinned oracle restatement of
  lz4.py:51-114.
- LZ4, fast mode (exact=False; vdi_lz4_compress, a chunk-parallel parse):
  parity is the transport's own property (test_acceptance.py A6): the
  reference decoder (oracle.lz4_decompress, the pinned restatement of
  lz4.py:117-168) returns the input exactly, and the block respects the
  format's end-of-block rules.
- validate_vdi: the reference's InvariantViolation messages on 13 cases.
"""

import hashlib

import numpy as np
import pytest

import golden_io as gio

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import codec, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200.camera import Camera  # noqa: E402
from paper_2206_08660_b200.vdi import InvariantViolation, validate_vdi  # noqa: E402
from oracle import oracle  # noqa: E402


def _fixture(src):
    counts, segs, grid, gen, aabb = gio.fixture_vdi(src)
    p, vp = gen["gen_pose"], gen["gen_viewport"]
    cam = Camera(position=tuple(p[0:3]), orientation=tuple(p[3:7]), fov_y=float(p[7]),
                 near=float(p[8]), far=float(p[9]), viewport=(int(vp[0]), int(vp[1])))
    h, w, n_sg, _ = segs.shape
    gz, gy, gx = grid.shape
    vdi = vb.Vdi(w, h, n_sg, counts, segs, cam, aabb)
    return vdi, vb.AccelGrid((gx, gy, gz), grid, cam.near, cam.far), gen


def _check_block(comp, raw):
    """Decodes with the reference decoder; end-of-block rules of the format."""
    assert oracle.lz4_decompress(comp, len(raw)) == raw
    assert len(comp) <= len(raw) + len(raw) // 255 + 16


def test_encode_vdi_matches_reference():
    g = gio.load("codec")
    for k, src in enumerate(str(t) for t in g["vdi_tags"]):
        vdi, grid, gen = _fixture(src)
        raw = codec.encode_vdi(vdi, grid)
        assert hashlib.sha256(raw).hexdigest() == str(g[f"v{k}_raw_sha256"]), src
        ref = g[f"v{k}_lz4"].tobytes()
        assert codec.compress(raw) == ref, src  # the reference's own block
        comp2, n = codec.compress_vdi(vdi, grid)
        assert n == len(raw) and comp2 == ref, src
        _check_block(codec.compress(raw, exact=False), raw)
        comp3, n3 = codec.compress_vdi(vdi, grid, exact=False)
        assert n3 == len(raw)
        _check_block(comp3, raw)


def test_lz4_reference_vectors():
    """Exact mode reproduces the reference's blocks of every byte vector
    (sizes around the 12-byte match limit and the 5-byte literal tail, runs,
    255-run length extensions, random data); fast mode round-trips them."""
    g = gio.load("codec")
    for k in range(int(g["n_bytes_cases"])):
        raw = g[f"b{k}_in"].tobytes()
        for exact in (True, False):
            comp = codec.compress(raw, exact=exact)
            if not raw:
                assert comp == b""
                continue
            _check_block(comp, raw)
            if exact:
                assert comp == g[f"b{k}_lz4"].tobytes(), k


@pytest.mark.parametrize("n", [12, 13, 17, 32767, 32768, 32769, 65536 + 5, 3 * 32768 + 7, 300001])
def test_lz4_chunk_boundaries(n):
    rng = np.random.default_rng(n)
    words = [rng.integers(0, 256, int(k), dtype=np.uint8).tobytes()
             for k in rng.integers(4, 64, 40)]
    raw = b"".join(words[int(i)] for i in rng.integers(0, 40, n // 4 + 1))[:n]
    raw = raw[:n // 2] + b"\x00" * (n - n // 2)
    comp = codec.compress(raw)
    assert comp == oracle.lz4_compress(raw)
    _check_block(codec.compress(raw, exact=False), raw)


@pytest.mark.parametrize("shift", [1, 2, 3])
def test_lz4_unaligned_source(shift):
    """The C ABI takes any device pointer: windows of an unaligned source are
    assembled from aligned words (csrc/vdi_codec.cu window_load/value)."""
    rng = np.random.default_rng(shift)
    words = [rng.integers(0, 256, int(k), dtype=np.uint8).tobytes()
             for k in rng.integers(4, 64, 40)]
    n = 4 * 32768 + 1001
    raw = b"".join(words[int(i)] for i in rng.integers(0, 40, n // 4 + 1))[:n]
    buf = dv.to_device(np.frombuffer(b"\x55" * shift + raw + b"\xaa" * 3, dtype=np.uint8))
    for exact in (True, False):
        dst, out_len = codec.compress_device(buf[shift:shift + n], n, exact=exact)
        m = int(dv.to_host(out_len)[0])
        comp = dv.to_host(dst[:m]).tobytes()
        _check_block(comp, raw)
        if exact:
            assert comp == oracle.lz4_compress(raw)


def test_lz4_device_length_clamped_to_capacity():
    """A device length above n_max compresses the first n_max bytes (the
    workspace and dst are sized for n_max; include/vdi_b200.h)."""
    rng = np.random.default_rng(5)
    raw = (rng.integers(0, 4, 70000, dtype=np.uint8) * 17).tobytes()
    n_max = 65536 + 77
    src = dv.to_device(np.frombuffer(raw, dtype=np.uint8))
    n_dev = torch.tensor([len(raw) + 12345], dtype=torch.int64, device="cuda")
    for exact in (True, False):
        dst, out_len = codec.compress_device(src, n_max, n_dev, exact=exact)
        m = int(dv.to_host(out_len)[0])
        comp = dv.to_host(dst[:m]).tobytes()
        _check_block(comp, raw[:n_max])
        if exact:
            assert comp == oracle.lz4_compress(raw[:n_max])


def test_lz4_ratio_close_to_reference():
    """Chunk-parallel parsing loses little against the serial parse."""
    g = gio.load("codec")
    for k in range(int(g["n_bytes_cases"])):
        raw = g[f"b{k}_in"].tobytes()
        if len(raw) < 4096:
            continue
        ours = len(codec.compress(raw, exact=False))
        ref = len(g[f"b{k}_lz4"].tobytes())
        assert ours <= ref * 1.05 + 64, (k, ours, ref)


@pytest.mark.parametrize("cfg", ["C1", "C3"])
def test_compress_vdi_full_size(cfg):
    vol, tf, gcam, rcam, n_sg = synth.config(cfg)
    vdi, grid = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg))
    comp, n = codec.compress_vdi(vdi, grid)
    fast, n2 = codec.compress_vdi(vdi, grid, exact=False)
    cam = vdi.gen_camera
    ref_raw = oracle.encode_vdi(vdi.width, vdi.height, n_sg, vdi.counts, vdi.segs,
                                (*cam.position, *cam.orientation, cam.fov_y, cam.near, cam.far),
                                vdi.volume_aabb, grid.counts)
    assert n == len(ref_raw) and n2 == n
    assert comp == oracle.lz4_compress(ref_raw)  # the reference's serial parse
    assert oracle.lz4_decompress(fast, n) == ref_raw
    validate_vdi(vdi)


def test_validate_messages_match_reference():
    g = gio.load("codec")
    vdi0, _, _ = _fixture("random_vdi:1")
    for k, msg in enumerate(str(m) for m in g["val_messages"]):
        v = vb.Vdi(8, 6, vdi0.n_sg, g[f"val{k}_counts"], g[f"val{k}_segs"], vdi0.gen_camera,
                   vdi0.volume_aabb)
        if msg == "":
            validate_vdi(v)
        else:
            with pytest.raises(InvariantViolation) as e:
                validate_vdi(v)
            assert str(e.value) == msg, k


def test_decode_vdi_matches_reference_arrays():
    """vdi.py:162-210 on the device: reference VDI1 bytes (the golden LZ4
    blocks decompressed by the reference decoder) decode to the fixture's
    counts, segments (zero past each count) and grid, and re-encode to the
    same bytes; the reference's error cases raise its exceptions."""
    from paper_2206_08660_b200.vdi import InvariantViolation
    g = gio.load("codec")
    for k, src in enumerate(str(t) for t in g["vdi_tags"]):
        vdi0, grid0, gen = _fixture(src)
        raw = oracle.lz4_decompress(g[f"v{k}_lz4"].tobytes(), int(g[f"v{k}_raw_len"]))
        vdi, grid = codec.decode_vdi(raw)
        assert np.array_equal(vdi.counts, vdi0.counts), src
        assert np.array_equal(vdi.segs.view(np.uint32), vdi0.segs.view(np.uint32)), src
        assert np.array_equal(grid.counts, grid0.counts), src
        assert codec.encode_vdi(vdi, grid) == raw, src
    vdi0, grid0, _ = _fixture("sphere64_u8")
    raw = codec.encode_vdi(vdi0, grid0)
    with pytest.raises(codec.BadMagic):
        codec.decode_vdi(b"XDI1" + raw[4:])
    with pytest.raises(codec.VersionMismatch):
        codec.decode_vdi(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(codec.TruncatedStream):
        codec.decode_vdi(raw[:-1])
    with pytest.raises(codec.TruncatedStream):
        codec.decode_vdi(raw + b"\x00")
    bad = bytearray(raw)
    w = int.from_bytes(raw[8:12], "little")
    n_sg = int.from_bytes(raw[16:20], "little")
    bad[160:162] = (n_sg + 1).to_bytes(2, "little")  # list (0,0) count > n_sg
    bad = bytes(bad) + b"\x00" * 24 * (n_sg + 1 - int.from_bytes(raw[160:162], "little"))
    with pytest.raises(InvariantViolation) as e:
        codec.decode_vdi(bad)
    assert str(e.value) == f"list (0,0) count {n_sg + 1} > n_sg {n_sg}"  # vdi.py:199-201
    del w
