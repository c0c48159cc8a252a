"""C5 (BASELINE configs[4]): Richtmyer-Meshkov-shaped 2048 x 2048 x 1920 u8
volume (synthesised on the device), 3840 x 2160, n_sg 40, render at 15 deg,
on one B200 (the 8-GPU bricked placement is exercised by tests/test_shard*).

Generation is checked on every list (device validate_vdi, count budget,
pass bound) and against the oracle on every 8th 16-row band (17 bands, 272
rows, 1.04 M rays: the oracle reads the raw u8 voxels, normalised exactly as
volume.py:48-50); the render at 15 deg is checked against the oracle per
pixel on the same rows, including the lists-visited /
supersegments-intersected / lists-searched counters.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import _capi, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200.raycast import launch_render  # noqa: E402
import fullframe as ff  # noqa: E402
from oracle import oracle, parity  # noqa: E402

# every 8th 16-row band of the 2160 rows (SURVEY 8(d)'s deterministic subset)
ROWS = np.concatenate([np.arange(16 * b, 16 * b + 16) for b in range(0, 135, 8)])


def rows_aos(vdi, rows):
    """(len(rows), W, n_sg, 6) AoS of the device VDI's rows (no full copy)."""
    d = vdi.device()
    w, n = vdi.width, vdi.n_sg
    idx = torch.as_tensor(rows, device=d.segs.device)
    soa = d.segs.view(-1, w, d.segs.shape[1]).index_select(0, idx).reshape(len(rows) * w, -1)
    aos = torch.empty((len(rows) * w, n * 6), dtype=torch.float32, device=soa.device)
    _capi.check(_capi.load().vdi_segs_to_aos(dv.ptr(soa), dv.ptr(aos), len(rows) * w, n,
                                             dv.stream_handle()))
    return dv.to_host(d.counts.index_select(0, idx)), dv.to_host(aos).reshape(len(rows), w, n, 6)


@pytest.fixture(scope="module")
def c5():
    vol, tf, gcam, rcam, n_sg = synth.config("C5")
    params = vb.GenParams(n_sg=n_sg)
    vdi, grid, st = vb.generate_vdi(vol, tf, gcam, params, with_stats=True)
    return vol, tf, gcam, rcam, n_sg, params, vdi, grid, st


def test_c5_volume_deterministic(c5):
    vol = c5[0]
    again = synth.rm_like()
    assert torch.equal(vol.device_data, again.device_data)
    frac = float((vol.device_data > 0).float().mean())
    assert 0.1 < frac < 0.6, frac


def test_c5_generation(c5):
    vol, tf, gcam, rcam, n_sg, params, vdi, grid, st = c5
    vb.validate_vdi(vdi)
    assert int(vdi.device().counts.max()) <= n_sg and st.passes.max() <= 23
    delta, step, lref = params.resolve(vol)
    w, h = gcam.viewport
    ref = oracle.generate(vol.data, tf.lut, gcam.proj_view(), gcam.inv_proj_view(),
                          np.asarray(gcam.position), vol.aabb, w, h, n_sg, delta,
                          params.epsilon, params.gamma_init, step, lref, rows=ROWS,
                          compact=True)
    counts, segs = rows_aos(vdi, ROWS)
    blk = parity.generation(ref, counts, segs, st.passes[ROWS], st.samples[ROWS],
                            st.gammas[ROWS])
    ff.record("C5/gen_band8", blk)
    assert blk["rays"] == len(ROWS) * w
    assert blk["ok"], blk
    assert blk["counts_equal_frac"] == 1.0 and blk["segs_bit_exact"], blk
    assert blk["passes_equal"] and blk["samples_equal"] and blk["gammas_bit_exact"], blk


def test_c5_render(c5):
    psutil = pytest.importorskip("psutil")
    if psutil.virtual_memory().available < 40 << 30:
        pytest.skip("the oracle render needs the full 8 GB AoS VDI on the host")
    vol, tf, gcam, rcam, n_sg, params, vdi, grid, st = c5
    ow, oh = rcam.viewport
    image = torch.empty((oh, ow, 4), dtype=torch.float64, device="cuda")
    pp = [torch.empty((oh, ow), dtype=torch.int32, device="cuda") for _ in range(3)]
    launch_render(vdi, grid, rcam, vb.RenderOptions(), image, per_pixel=pp)
    img = dv.to_host(image)
    lv, si, ls = (dv.to_host(x) for x in pp)
    ref = oracle.render(vdi.segs, vdi.counts, gcam.proj_view(), gcam.inv_proj_view(), vol.aabb,
                        rcam.inv_proj_view(), np.asarray(rcam.position), ow, oh, grid.counts,
                        gcam.near, gcam.far, rows=ROWS)
    blk = parity.render(ref, img, lv, si, ls, rows=ROWS)
    ff.record("C5/render15_band8", blk)
    assert blk["ok"], blk
