"""Time render_dvr's kernel (vdi_dvr_launch) on a config, device resident.

    python tools/bench_dvr.py --config C3 [--reps 10] [--oracle-rows 8]

Prints one JSON line per view (generation view and render view of the
config): kernel ms (CUDA events, median over reps, 256 MiB L2 flush
between reps), Mrays/s, executed samples, and the algorithmic-bytes roofline
B_dvr = 32 S + 32 P (the reference reads the 8 f32 taps of Volume.normalized
per sample and writes an f64 RGBA pixel) against the
measured copy bandwidth. With --oracle-rows the oracle (CPU port of
dvr.py:21-89, OpenMP on all host cores) is timed on that many evenly spaced
rows and extrapolated per ray, as the CPU baseline.
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

from paper_2206_08660_b200 import _capi, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200.dvr import launch_dvr, resolve_steps  # noqa: E402


def peak_gbps():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C3")
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--oracle-rows", type=int, default=0)
    p.add_argument("--no-cells", action="store_true")
    a = p.parse_args()
    vol, tf, gcam, rcam, _ = synth.config(a.config)
    vol_dev, vt = dv.upload_volume(vol)
    lut = dv.upload_lut(tf.lut)
    bricks = dv.volume_bricks(vol_dev, vt, vol.dims)
    cells = (dv.volume_cells(vol_dev, vt, vol.dims)
             if dv.use_cells(vt, vol.dims) and not a.no_cells else None)
    step, lref = resolve_steps(vol, None, None)
    ws = torch.empty(_capi.DVR_WORKSPACE_BYTES, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    peak, peak_kind = peak_gbps()
    for tag, cam in (("gen_view", gcam), ("render_view", rcam)):
        w, h = cam.viewport
        img = torch.empty((h, w, 4), dtype=torch.float64, device="cuda")
        sums = torch.zeros(1, dtype=torch.int64, device="cuda")
        smp = torch.empty((h, w), dtype=torch.int32, device="cuda")

        def run(samples=None, stat=None):
            launch_dvr(vol_dev, vt, vol.dims, lut, cam, vol.aabb, step, lref, 0.999,
                       (0.0, 0.0, 0.0, 1.0), img, ws, samples=samples, stat_sums=stat,
                       bricks=bricks, ess_max=dv.ess_threshold(tf.lut), cells=cells)

        run(smp, sums)
        torch.cuda.synchronize()
        S = int(sums.item())
        times = []
        for _ in range(a.reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        P = w * h
        B = 32 * S + 32 * P
        line = {"tool": "bench_dvr", "config": a.config, "view": tag, "viewport": [w, h],
                "voxel": vt + ("+cells" if cells is not None else ""), "ms": ms,
                "mrays_s": P / ms / 1e3, "samples": S, "gsamples_s": S / ms / 1e6,
                "roofline": {"bound": "hbm", "algorithmic_bytes": B,
                             "achieved": B / ms / 1e6, "peak": peak, "peak_kind": peak_kind,
                             "unit": "GB/s", "frac": B / ms / 1e6 / peak}}
        if a.oracle_rows:
            sys.path.insert(0, ROOT)
            from oracle import oracle
            rows = np.linspace(0, h - 1, a.oracle_rows).round().astype(np.int32)
            t0 = time.perf_counter()
            ref = oracle.dvr(vol.normalized, tf.lut, cam.proj_view(), cam.inv_proj_view(),
                             np.asarray(cam.position), vol.aabb, w, h, step, lref, rows=rows)
            dt = time.perf_counter() - t0
            host = dv.to_host(img)
            line["cpu_baseline"] = {"mrays_s": len(rows) * w / dt / 1e6,
                                    "cores": oracle.max_threads(), "kind": "port",
                                    "sample": f"{len(rows)} evenly spaced rows ({dt:.2f} s)"}
            line["oracle_max_abs_diff"] = float(np.abs(host[rows] - ref[rows]).max())
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
