"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes metrics)
into per-kernel totals for the first generate+render step of the capture.

usage: python tools/summarize_launches.py launches.csv out.json [command string]
"""
import csv
import json
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
iN, iM, iV, iI = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
launches = OrderedDict()
for r in rows[1:]:
    d = launches.setdefault(int(r[iI]), {"kernel": r[iN].split("(")[0]})
    d[r[iM]] = float(r[iV])
# first step: from the first gen_sample launch up to and including the first render
ids = sorted(launches)
start = next(i for i in ids if "gen_sample" in launches[i]["kernel"]) - 1  # + fill_inv
end = next(i for i in ids if "render_kernel" in launches[i]["kernel"])
step = [launches[i] for i in ids if start <= i <= end]
phases = OrderedDict()
for l in step:
    k = l["kernel"].replace("void ", "").replace("vdi::", "").split("<")[0]
    p = phases.setdefault(k, {"launches": 0, "ms": 0.0, "dram_read": 0.0, "dram_write": 0.0})
    p["launches"] += 1
    p["ms"] += l.get("gpu__time_duration.sum", 0.0) / 1e6
    p["dram_read"] += l.get("dram__bytes_read.sum", 0.0)
    p["dram_write"] += l.get("dram__bytes_write.sum", 0.0)
gen = [p for k, p in phases.items() if k.startswith("gen_") or k == "fill_inv_kernel"]
out = {
    "source": sys.argv[1],
    "command": sys.argv[3] if len(sys.argv) > 3 else None,
    "note": "ncu --clock-control none, cold-cache serialised launches; compare shares",
    "phases": phases,
    "gen_dram_bytes_per_launch": sum(p["dram_read"] + p["dram_write"] for p in gen),
    "gen_ms": sum(p["ms"] for p in gen),
}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps({k: out[k] for k in ("gen_dram_bytes_per_launch", "gen_ms")}))
