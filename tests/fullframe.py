"""Shared helpers of the full-frame parity tests (C3, C4, C5 at BASELINE
sizes): the B200 VDI rows as host AoS, the render with per-pixel counters,
and the oracle runs on the same inputs."""

from __future__ import annotations

import json
import os

import numpy as np

from oracle import oracle, parity

PROFILES = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")


def vol_for_oracle(vol):
    """The raw u8 voxels when the volume is u8 (the oracle normalises them
    exactly as volume.py:48-50), else R's f32 `normalized`."""
    return vol.data if vol.voxel_type == "u8" else vol.normalized


def oracle_generate(vol, tf, cam, params, rows=None):
    delta, step, lref = params.resolve(vol)
    w, h = cam.viewport
    return oracle.generate(vol_for_oracle(vol), tf.lut, cam.proj_view(), cam.inv_proj_view(),
                           np.asarray(cam.position), vol.aabb, w, h, params.n_sg, delta,
                           params.epsilon, params.gamma_init, step, lref, rows=rows,
                           compact=rows is not None)


def oracle_render(counts, segs, grid_counts, vol, gcam, cam, rows=None):
    ow, oh = cam.viewport
    return oracle.render(segs, counts, gcam.proj_view(), gcam.inv_proj_view(), vol.aabb,
                         cam.inv_proj_view(), np.asarray(cam.position), ow, oh, grid_counts,
                         gcam.near, gcam.far, rows=rows)


def gpu_render(vdi, grid, cam, opts=None):
    """B200 render with per-pixel counters: (image, lists_visited,
    segs_intersected, lists_searched) on the host."""
    import paper_2206_08660_b200 as vb
    from paper_2206_08660_b200 import device as dv
    from paper_2206_08660_b200.raycast import launch_render
    t = dv.torch()
    ow, oh = cam.viewport
    image = t.empty((oh, ow, 4), dtype=t.float64, device="cuda")
    pp = [t.empty((oh, ow), dtype=t.int32, device="cuda") for _ in range(3)]
    launch_render(vdi, grid, cam, opts or vb.RenderOptions(), image, per_pixel=pp)
    return (dv.to_host(image),) + tuple(dv.to_host(x) for x in pp)


def rows_aos(vdi, rows):
    """(counts, AoS segs) of the device VDI's `rows`, without a full copy."""
    from paper_2206_08660_b200 import _capi
    from paper_2206_08660_b200 import device as dv
    t = dv.torch()
    d = vdi.device()
    w, n = vdi.width, vdi.n_sg
    idx = t.as_tensor(np.asarray(rows), device=d.segs.device)
    soa = d.segs.view(-1, w, d.segs.shape[1]).index_select(0, idx).reshape(len(rows) * w, -1)
    aos = t.empty((len(rows) * w, n * 6), dtype=t.float32, device=soa.device)
    _capi.check(_capi.load().vdi_segs_to_aos(dv.ptr(soa), dv.ptr(aos), len(rows) * w, n,
                                             dv.stream_handle()))
    return (dv.to_host(d.counts.index_select(0, idx)),
            dv.to_host(aos).reshape(len(rows), w, n, 6))


def record(name: str, block: dict) -> None:
    """Print the parity block (pytest -s shows it; the GPU scripts keep the
    log under profiles/)."""
    print(f"PARITY {name} {json.dumps(block, sort_keys=True)}", flush=True)


__all__ = ["parity", "oracle_generate", "oracle_render", "gpu_render", "rows_aos", "record",
           "vol_for_oracle"]
