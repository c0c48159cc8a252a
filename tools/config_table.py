"""Results table over the BASELINE configs (C1..C5) on one B200: generation
and render (device resident, CUDA events, median of --reps, 256 MiB L2 flush
before each step), their algorithmic-byte rooflines (BASELINE.md section 4:
B_gen = 32 S + N (4 + 24 n_sg) + 4 g, B_ren = 4 L + 8 L_s + 24 K + 32 P, with
S / L / L_s / K the kernels' exact counters), and the CPU port of the
reference kernels (oracle, OpenMP on all host cores) on evenly spaced rows of
both passes, extrapolated per ray. One JSON line per config, then a
markdown table.

    python tools/config_table.py [--configs C1,C2,C3,C4,C5] [--reps 3] [--cpu-rows 6]
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

from paper_2206_08660_b200 import shard, synth  # noqa: E402
from paper_2206_08660_b200.generate import GenParams  # noqa: E402


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", default="C1,C2,C3,C4,C5")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--cpu-rows", type=int, default=6)
    a = p.parse_args()
    pk = peak()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    rows_out = []
    for cfg in a.configs.split(","):
        vol, tf, gcam, rcam, n_sg = synth.config(cfg)
        params = GenParams(n_sg=n_sg)
        pipe = shard.Pipeline(vol, tf, gcam, rcam, params)
        pipe.step()
        torch.cuda.synchronize()
        evs = []
        for _ in range(a.reps):
            flush.fill_(1)
            evs.append(pipe.step(timed=True))
        g_ms = float(np.median([e["gen"] + e["grid"] for e in evs]))
        r_ms = float(np.median([e["render"] for e in evs]))
        prep = float(np.median([e["prep"] for e in evs]))
        S = pipe.samples_executed()
        L, K, Ls = pipe.exact_render_stats()
        w, h = gcam.viewport
        ow, oh = rcam.viewport
        gx, gy, gz = pipe.grid_dims
        b_gen = 32 * S + w * h * (4 + 24 * n_sg) + 4 * gx * gy * gz
        b_ren = 4 * L + 8 * Ls + 24 * K + 32 * ow * oh
        line = {"config": cfg, "viewport": [w, h], "n_sg": n_sg, "prep_ms": prep,
                "gen_ms": g_ms, "gen_mrays_s": w * h / g_ms / 1e3, "samples": S,
                "gen_frac": b_gen / (g_ms * 1e-3) / 1e9 / pk,
                "render_ms": r_ms, "render_mrays_s": ow * oh / r_ms / 1e3,
                "render_fps": 1e3 / r_ms, "render_frac": b_ren / (r_ms * 1e-3) / 1e9 / pk,
                "lists_visited": L, "segs_intersected": K, "lists_searched": Ls}
        if a.cpu_rows:
            from oracle import oracle
            rows = np.unique(np.linspace(0, h - 1, a.cpu_rows).round().astype(np.int64))
            delta, step, lref = params.resolve(vol)
            vdata = vol.data if vol.voxel_type == "u8" else vol.normalized
            t0 = time.perf_counter()
            oracle.generate(vdata, tf.lut, gcam.proj_view(), gcam.inv_proj_view(),
                            np.asarray(gcam.position), vol.aabb, w, h, n_sg, delta,
                            params.epsilon, params.gamma_init, step, lref, rows=rows,
                            compact=True)
            tg = time.perf_counter() - t0
            counts, segs, grid = pipe.host_vdi()
            orow = np.unique(np.linspace(0, oh - 1, a.cpu_rows).round().astype(np.int64))
            t0 = time.perf_counter()
            oracle.render(segs, counts, gcam.proj_view(), gcam.inv_proj_view(), vol.aabb,
                          rcam.inv_proj_view(), np.asarray(rcam.position), ow, oh, grid,
                          gcam.near, gcam.far, rows=orow)
            tr = time.perf_counter() - t0
            line["cpu"] = {"gen_mrays_s": len(rows) * w / tg / 1e6,
                           "render_mrays_s": len(orow) * ow / tr / 1e6,
                           "cores": oracle.max_threads(), "kind": "port",
                           "sample": f"{len(rows)} gen rows ({tg:.1f} s), {len(orow)} render "
                                     f"rows ({tr:.2f} s)"}
        print(json.dumps(line), flush=True)
        rows_out.append(line)
        del pipe, vol
        torch.cuda.empty_cache()
    print("\n| config | gen ms | gen Mrays/s | gen % roofline | render ms | render Mrays/s | "
          "render % roofline | CPU gen / render Mrays/s (cores) |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows_out:
        c = r.get("cpu", {})
        cpu = (f"{c['gen_mrays_s']:.3f} / {c['render_mrays_s']:.2f} ({c['cores']})"
               if c else "—")
        print(f"| {r['config']} | {r['gen_ms']:.2f} | {r['gen_mrays_s']:.1f} | "
              f"{100 * r['gen_frac']:.1f} | {r['render_ms']:.3f} | {r['render_mrays_s']:.0f} | "
              f"{100 * r['render_frac']:.1f} | {cpu} |")


if __name__ == "__main__":
    main()
