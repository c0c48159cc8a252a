"""Markdown table of the key `ncu --set full` metrics of every kernel in a
report (one column per launch):

    python tools/ncu_summary.py gpurun_out/r02_gen_phases.ncu-rep
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("Duration", "duration"),
    ("Registers Per Thread", "registers / thread"),
    ("Theoretical Occupancy", "theoretical occupancy %"),
    ("Achieved Active Warps Per SM", "achieved warps / SM"),
    ("Compute (SM) Throughput", "compute (SM) throughput %"),
    ("Issued Ipc Active", "issued IPC (active)"),
    ("Issue Slots Busy", "issue slots busy %"),
    ("Warp Cycles Per Issued Instruction", "warp cycles / issued inst"),
    ("Avg. Active Threads Per Warp", "active threads / warp"),
    ("Executed Instructions", "warp instructions"),
    ("DRAM Throughput", "DRAM throughput % of peak"),
    ("L1/TEX Hit Rate", "L1 hit %"),
    ("L2 Hit Rate", "L2 hit %"),
    ("SM Active Cycles", "SM active cycles"),
    ("Elapsed Cycles", "elapsed cycles"),
]


def short(name):
    m = re.search(r"(\w+)(<[^>]*>)?\(", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:40]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    iI, iK, iS, iM, iU, iV = (h.index(x) for x in ("ID", "Kernel Name", "Section Name",
                                                  "Metric Name", "Metric Unit", "Metric Value"))
    launches = {}
    for r in rows[1:]:
        if len(r) <= iV:
            continue
        d = launches.setdefault(r[iI], {"name": r[iK]})
        key = r[iM]
        if key == "Memory Throughput" and r[iU] != "Gbyte/s":
            continue
        d.setdefault(key, (r[iV], r[iU]))
    # warp-state stall breakdown is in the raw page; keep the table to the details page
    ids = list(launches)
    print("| metric | " + " | ".join(f"#{i} {short(launches[i]['name'])}" for i in ids) + " |")
    print("|---|" + "---|" * len(ids))
    for k, label in KEYS:
        vals = []
        for i in ids:
            v = launches[i].get(k)
            vals.append(f"{v[0]} {v[1]}".strip() if v and k in ("Duration",) else (v[0] if v else ""))
        print(f"| {label} | " + " | ".join(vals) + " |")
    # stall reasons (PC samples) from the raw page, top 5 per launch
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hh = rr[0]
    tops = []
    for r in rr[2:]:
        d = dict(zip(hh, r))
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
              for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:5]
        tops.append(", ".join(f"{k} {100 * v / tot:.1f} %" for k, v in top))
    print("| stall reasons (PC samples) | " + " | ".join(tops) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
