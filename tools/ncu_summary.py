"""Key numbers of one ncu --set full report: speed of light, occupancy, warp
state, stall reasons, DRAM traffic, and the hottest SASS lines by stall samples.

usage: python tools/ncu_summary.py report.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 12


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
raw = dict(zip(h, v))
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
for k in keys:
    if k in raw:
        print(f"{k} = {raw[k]}")
st = [(k, float(val)) for k, val in raw.items()
      if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
      and val.replace(".", "", 1).isdigit()]
st.sort(key=lambda x: -x[1])
print("stalls per issue:", ", ".join(f"{k[34:-23]}={x:.2f}" for k, x in st[:8]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh = src[1]
data = src[2:]
iA, iS, iT = hh.index("Address"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iT] or 0) for r in data)
print(f"stall samples: {tot:.0f}; hottest SASS:")
reasons = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
for i in sorted(range(len(data)), key=lambda i: -float(data[i][iT] or 0))[:top_n]:
    r = data[i]
    why = max(reasons, key=lambda c: float(r[hh.index(c)] or 0))
    print(f"  {r[iA][-5:]} {100 * float(r[iT]) / tot:5.1f}% {why:22s} {r[iS].strip()[:70]}")
