"""Time render_preview's kernels (vdi_preview_launch + upsample) on a
config, device resident: generate the config's VDI, then preview it from the
render view at several (d_i, d_r). Prints one JSON line per setting with
the kernel time (CUDA events, median), samples and samples/s. With
--oracle the CPU port (preview.py:49-205 in C, OpenMP) is timed on the same
frame for the CPU baseline.

    python tools/bench_preview.py --config C3 [--reps 5] [--oracle]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import _capi, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200.camera import Camera  # noqa: E402
from paper_2206_08660_b200.preview import (PreviewParams, low_res_viewport,  # noqa: E402
                                           preview_args, upsample_device)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C3")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--oracle", action="store_true")
    a = p.parse_args()
    vol, tf, gcam, rcam, n_sg = synth.config(a.config)
    vdi, grid = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg))
    disp = rcam.viewport
    for d_i, d_r in ((1.0, 1.0), (1.0, 0.25), (0.5, 0.5), (0.25, 1.0)):
        params = PreviewParams(d_i=d_i, d_r=d_r, display=disp)
        lw, lh = low_res_viewport(params)
        low = Camera(position=rcam.position, orientation=rcam.orientation, fov_y=rcam.fov_y,
                     near=rcam.near, far=rcam.far, viewport=(lw, lh))
        image = torch.empty((lh, lw, 4), dtype=torch.float64, device="cuda")
        ws = torch.empty(_capi.PREVIEW_WORKSPACE_BYTES, dtype=torch.uint8, device="cuda")
        sums = torch.zeros(1, dtype=torch.int64, device="cuda")
        gx, gy, gz = grid.dims
        cells = torch.empty((gz, gy, gx), dtype=torch.int64, device="cuda")
        L = _capi.load()

        def run(stat=None, cs=None):
            args = preview_args(vdi.device(), vdi.n_sg, vdi.width, vdi.height, vdi.gen_camera,
                                vdi.volume_aabb, grid.device(), grid.dims, grid.near,
                                grid.far, low, d_r, 0.999, (0.0, 0.0, 0.0, 1.0), image, ws,
                                cs, stat)
            _capi.check(L.vdi_preview_launch(args, dv.stream_handle()))
            return upsample_device(image, *disp)

        run(sums, cells)
        torch.cuda.synchronize()
        S = int(sums.item())
        times = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        line = {"tool": "bench_preview", "config": a.config, "d_i": d_i, "d_r": d_r,
                "low_res": [lw, lh], "display": list(disp), "ms": ms, "samples": S,
                "gsamples_s": S / ms / 1e6, "fps": 1e3 / ms}
        if a.oracle:
            from oracle import oracle
            t0 = time.perf_counter()
            oracle.preview_lowres(vdi.segs, vdi.counts, gcam.proj_view(), gcam.inv_proj_view(),
                                  vol.aabb, low.inv_proj_view(), np.asarray(low.position),
                                  lw, lh, grid.counts, gcam.near, gcam.far, d_r)
            dt = time.perf_counter() - t0
            line["cpu_baseline"] = {"ms": dt * 1e3, "cores": oracle.max_threads(),
                                    "kind": "port", "sample": "the whole frame"}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
