"""One-screen summary of an ncu report (all kernels in it): duration, SOL,
IPC, occupancy, active threads per warp, cache hit rates, DRAM bytes, top
stall reasons. usage: python tools/ncu_brief.py X.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = {
    "Duration": "duration", "Compute (SM) Throughput": "sm_sol", "Memory Throughput": "mem_sol",
    "DRAM Throughput": "dram_sol", "Executed Ipc Active": "ipc",
    "Achieved Occupancy": "occupancy", "Registers Per Thread": "regs",
    "Avg. Active Threads Per Warp": "threads_per_warp", "L1/TEX Hit Rate": "l1_hit",
    "L2 Hit Rate": "l2_hit", "Warp Cycles Per Issued Instruction": "cpi",
}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    iK, iN, iV, iU = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    iI = h.index("ID")
    kern = {}
    for r in rows[1:]:
        if r[iN] in WANT:
            kern.setdefault((r[iI], r[iK][:40]), {})[WANT[r[iN]]] = f"{r[iV]} {r[iU]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh = rr[0]
    for r in rr[2:]:
        key = (r[hh.index("ID")], r[hh.index("Kernel Name")][:40])
        d = kern.setdefault(key, {})
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if m in hh:
                d[m.split(".")[0]] = r[hh.index(m)] + " " + rr[1][hh.index(m)]
    for (i, k), d in kern.items():
        print(f"[{i}] {k}")
        for kk, v in d.items():
            print(f"    {kk:18s} {v}")


if __name__ == "__main__":
    main(sys.argv[1])
