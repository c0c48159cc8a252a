"""Host-side logic of the drop-in API (no GPU): parameter validation with the
reference's errors, loud failure without a device, band maps, synth
determinism, the layout/validator helpers."""

import numpy as np
import pytest

import paper_2206_08660_b200 as vb
from paper_2206_08660_b200 import shard, synth
from paper_2206_08660_b200.vdi import default_grid_dims


def test_genparams_resolve_matches_reference_rules():
    # generate.py:38-50 and test_generate.py:253-265
    vol = vb.make_volume(np.zeros((4, 4, 4), np.uint8), "u8")
    with pytest.raises(ValueError):
        vb.GenParams(n_sg=0).resolve(vol)
    with pytest.raises(ValueError):
        vb.GenParams(epsilon=2.0).resolve(vol)
    assert vb.GenParams(n_sg=12).resolve(vol) == (1, 0.5, 0.5)
    assert vb.GenParams(n_sg=20).resolve(vol)[0] == 3
    assert vb.GenParams(n_sg=30).resolve(vol)[0] == 4
    assert vb.GenParams(n_sg=40).resolve(vol)[0] == 6
    assert vb.GenParams(n_sg=4, delta=9).resolve(vol)[0] == 3


def test_render_options_validation():
    with pytest.raises(ValueError):
        vb.RenderOptions(early_term_alpha=0.0)
    with pytest.raises(ValueError):
        vb.RenderOptions(early_term_alpha=1.5)
    vb.RenderOptions(early_term_alpha=1.0)


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    vol = synth.blobs(16)
    cam = synth.sweep_camera(vol, 0.0, (8, 8))
    with pytest.raises(RuntimeError):
        vb.generate_vdi(vol, synth.preset_tf("blobs"), cam, vb.GenParams(n_sg=4))


def test_volume_normalization_matches_reference_rule():
    data = np.arange(256, dtype=np.uint8).reshape(4, 4, 16)
    vol = vb.make_volume(data, "u8")
    assert vol.normalized.dtype == np.float32
    assert np.array_equal(vol.normalized, data.astype(np.float32) / np.float32(255.0))
    assert vol.normalized_is_derived


def test_default_grid_dims():
    assert default_grid_dims(1920, 1080) == (120, 67, 32)
    assert default_grid_dims(3840, 2160) == (240, 135, 32)
    assert default_grid_dims(8, 8) == (1, 1, 32)


@pytest.mark.parametrize("h,world", [(1080, 1), (1080, 2), (1080, 4), (1080, 8), (100, 3),
                                     (2160, 8), (16, 4)])
def test_band_partition_covers_rows_once(h, world):
    owned = np.concatenate([shard.band_rows(h, world, r) for r in range(world)])
    assert np.array_equal(np.sort(owned), np.arange(h))
    per = shard.rows_per_rank(h, world)
    assert all(shard.local_rows(h, world, r) <= per for r in range(world))
    st = shard.storage_rows(h, world)
    # a gathered buffer [world][per] holds every row exactly once
    assert len(np.unique(st)) == h and st.max() < world * per
    for r in range(world):
        rows = shard.band_rows(h, world, r)
        assert np.array_equal(st[rows], r * per + np.arange(len(rows)))


def test_synth_is_deterministic():
    a = synth.blobs(32)
    b = synth.blobs(32)
    assert np.array_equal(a.data, b.data)
    k1 = synth.kingsnake((64, 64, 50))
    k2 = synth.kingsnake((64, 64, 50))
    assert np.array_equal(k1.data, k2.data)
    assert k1.data.max() > 150 and (k1.data == 0).mean() > 0.3
