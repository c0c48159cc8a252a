"""FrameStream (overlapped H2D / kernels / D2H over a stream of volumes) gives,
frame by frame, exactly what the one-frame public API gives for that frame's
volume -- with alternating volumes, so a slot mix-up cannot go unnoticed."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200 import shard, synth  # noqa: E402
from paper_2206_08660_b200.stream import FrameStream  # noqa: E402
from paper_2206_08660_b200.volume import make_volume  # noqa: E402


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_stream_frames_match_single_frame_api(name):
    vol, tf, gcam, rcam, n_sg = synth.config(name)
    other = make_volume(np.ascontiguousarray(vol.data[::-1]), vol.voxel_type)  # same dims
    params = vb.GenParams(n_sg=n_sg)
    refs = []
    for v in (vol, other):
        vdi, grid = vb.generate_vdi(v, tf, gcam, params)
        img = vb.render_vdi(vdi, grid, rcam)
        refs.append((vdi.counts, vdi.segs, grid.counts, img.data))
    pipe = shard.Pipeline(vol, tf, gcam, rcam, params)
    fs = FrameStream(pipe)
    hosts = []
    for v in (vol, other):
        h = dv.pinned_numpy(v.data.shape, v.data.dtype)
        h[...] = v.data
        hosts.append(h)
    order = [0, 1, 0, 1, 1, 0]
    seen = []

    def check(r):
        c, s, g, im = refs[order[r.index]]
        h, w = c.shape
        assert np.array_equal(r.counts[:h], c)
        assert np.array_equal(r.segs[:h], s)
        assert np.array_equal(r.grid, g)
        oh = im.shape[0]
        assert np.array_equal(r.image[:oh], im)
        seen.append(r.index)

    n = fs.run([hosts[i] for i in order], on_result=check)
    assert n == len(order) and seen == list(range(len(order)))
    assert fs.h2d_bytes == vol.data.nbytes and fs.d2h_bytes > 0


def test_stream_packed_vdi1_matches_encode_vdi():
    """packed=True: each frame's VDI comes back as the VDI1 bytes of
    encode_vdi (vdi.py:141-159) of that frame's VDI, and decodes to it."""
    from paper_2206_08660_b200 import codec
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    other = make_volume(np.ascontiguousarray(vol.data[::-1]), vol.voxel_type)
    params = vb.GenParams(n_sg=n_sg)
    refs = []
    for v in (vol, other):
        vdi, grid = vb.generate_vdi(v, tf, gcam, params)
        img = vb.render_vdi(vdi, grid, rcam)
        refs.append((codec.encode_vdi(vdi, grid), vdi.counts, vdi.segs, grid.counts, img.data))
    pipe = shard.Pipeline(vol, tf, gcam, rcam, params)
    fs = FrameStream(pipe, packed=True)
    hosts = []
    for v in (vol, other):
        h = dv.pinned_numpy(v.data.shape, v.data.dtype)
        h[...] = v.data
        hosts.append(h)
    order = [1, 0, 0, 1]

    def check(r):
        raw, c, s, g, im = refs[order[r.index]]
        assert r.vdi1.tobytes() == raw
        dc, ds, dg = r.decode()
        assert np.array_equal(dc, c) and np.array_equal(ds, s) and np.array_equal(dg, g)
        assert np.array_equal(r.image[:im.shape[0]], im)

    assert fs.run([hosts[i] for i in order], on_result=check) == len(order)


@pytest.mark.parametrize("packed", [False, True])
def test_stream_in_flight_limit(packed):
    """At most two frames in flight: a third submit before a collect raises
    (its slots would overwrite the oldest frame's results), and a collect
    with nothing in flight raises; the two frames in flight stay correct."""
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    params = vb.GenParams(n_sg=n_sg)
    vdi, grid = vb.generate_vdi(vol, tf, gcam, params)
    pipe = shard.Pipeline(vol, tf, gcam, rcam, params)
    fs = FrameStream(pipe, packed=packed)
    h = dv.pinned_numpy(vol.data.shape, vol.data.dtype)
    h[...] = vol.data
    fs.submit(h)
    fs.submit(h)
    with pytest.raises(RuntimeError):
        fs.submit(h)
    for _ in range(2):
        r = fs.collect()
        c = r.decode()[0] if packed else r.counts
        assert np.array_equal(c, vdi.counts)
    with pytest.raises(RuntimeError):
        fs.collect()


def test_stream_rejects_bricked_pipeline():
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    pipe = shard.Pipeline(vol, tf, gcam, rcam, vb.GenParams(n_sg=n_sg), world=2, rank=0,
                          bricked=True)
    with pytest.raises(NotImplementedError):
        FrameStream(pipe)
    with pytest.raises(NotImplementedError):
        pipe.e2e(1)
