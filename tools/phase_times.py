"""Per-kernel time of one generate+render step from an ncu --csv launch list
(gpu__time_duration.sum): total ms per kernel name divided by the number of
steps in the capture (counted by render_kernel launches).

usage: python tools/phase_times.py launches.csv
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
iN, iM, iV = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value"))
tot = OrderedDict()
steps = 0
for r in rows[1:]:
    if r[iM] != "gpu__time_duration.sum":
        continue
    k = r[iN].split("(")[0].replace("void ", "").replace("vdi::", "").split("<")[0]
    if k == "render_kernel":
        steps += 1
    tot[k] = tot.get(k, 0.0) + float(r[iV]) / 1e6
steps = max(steps, 1)
print(" ".join(f"{k}={v / steps:.2f}" for k, v in tot.items() if v / steps > 0.05))
