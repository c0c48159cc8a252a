"""Per-kernel metrics of ONE pipeline step from an ncu --metrics CSV (the
tools/gpu/r02_metrics.sh capture of `tools/run_pipeline.py --config C --reps
2`: the second step's launches) -> profiles/<tag>_<cfg>_kernel_metrics.json,
which bench.py quotes in its roofline block (actual DRAM traffic, FP64 pipe
utilisation, warp execution efficiency per generation phase and render).

    python tools/ncu_metrics_json.py gpurun_out/r02_c3_metrics.csv C3 r02
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PHASES = ["brick_max", "cells", "fill_inv", "gen_setup", "gen_sample", "queue_", "gen_fill",
          "gen_bisect_wide", "gen_bisect", "gen_emit", "gen_fused", "grid_kernel", "grid_zmask",
          "list_ranges", "render_kernel"]
GEN = ("fill_inv", "gen_setup", "gen_sample", "queue_", "gen_fill", "gen_bisect_wide",
       "gen_bisect", "gen_emit", "gen_fused")


def phase_of(name):
    for p in PHASES:
        if p in name:
            return p
    return None


def main(path, cfg, tag):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    iK, iM, iV, iI = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("ID"))
    launches = {}
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        d = launches.setdefault(int(r[iI]), {"name": r[iK]})
        d[r[iM]] = float(r[iV].replace(",", ""))
    ids = sorted(launches)
    # the second step: from the second brick-maxima launch on
    starts = [i for i in ids if "brick_max" in launches[i]["name"]]
    first = starts[1] if len(starts) > 1 else ids[0]
    agg = {}
    for i in ids:
        if i < first:
            continue
        d = launches[i]
        ph = phase_of(d["name"])
        if ph is None:
            continue
        a = agg.setdefault(ph, {"launches": 0, "ms": 0.0, "dram_bytes": 0.0, "inst": 0.0,
                                "fp64_inst": 0.0, "_fp64w": 0.0, "_effw": 0.0, "_l2w": 0.0})
        t = d["gpu__time_duration.sum"] / 1e6
        a["launches"] += 1
        a["ms"] += t
        a["dram_bytes"] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        a["inst"] += d["sm__inst_executed.sum"]
        a["fp64_inst"] += d["sm__inst_executed_pipe_fp64.sum"]
        a["_fp64w"] += t * d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"]
        a["_effw"] += t * d["smsp__thread_inst_executed_per_inst_executed.ratio"] / 32.0
        a["_l2w"] += t * d["lts__t_sector_hit_rate.pct"]
    for a in agg.values():
        ms = max(a["ms"], 1e-12)
        a["fp64_pipe_pct"] = a.pop("_fp64w") / ms
        a["warp_exec_efficiency"] = a.pop("_effw") / ms
        a["l2_hit_pct"] = a.pop("_l2w") / ms
        a["dram_GBps"] = a["dram_bytes"] / (ms * 1e-3) / 1e9
    gen = [agg[p] for p in GEN if p in agg]
    commit = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                            capture_output=True, text=True).stdout.strip()
    out = {"config": cfg, "commit": commit,
           "source": f"{os.path.basename(path)}: ncu --metrics (time, DRAM bytes, FP64 pipe, "
                     "thread/warp, L2 hit) of tools/run_pipeline.py --config "
                     f"{cfg} --reps 2, second step; ncu times are serialised and cold-cache",
           "gen_dram_bytes": sum(a["dram_bytes"] for a in gen),
           "gen_ms_ncu": sum(a["ms"] for a in gen),
           "kernels": agg}
    dst = os.path.join(ROOT, "profiles", f"{tag}_{cfg.lower()}_kernel_metrics.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(dst)
    for p, a in agg.items():
        print(f"{p:14s} {a['ms']:8.3f} ms  DRAM {a['dram_bytes'] / 1e9:7.2f} GB "
              f"({a['dram_GBps']:7.0f} GB/s)  FP64 pipe {a['fp64_pipe_pct']:5.1f} %  "
              f"warp eff {a['warp_exec_efficiency']:5.2f}  L2 hit {a['l2_hit_pct']:5.1f} %")


if __name__ == "__main__":
    main(*sys.argv[1:4])
