"""Summarise an ncu SASS source page: hottest instructions with their top stall
reasons. usage: ncu -i X.ncu-rep --page source --csv --print-source=sass > s.csv;
python tools/sass_hot.py s.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


K = "Warp Stall Sampling (All Samples)"
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(f(d[K]) for d in data)
print(f"total samples {tot:.0f}, {len(data)} instructions")
agg = {s: sum(f(d[s]) for d in data) for s in stalls}
print("stalls:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in
                          sorted(agg.items(), key=lambda x: -x[1])[:8]))
idx = sorted(range(len(data)), key=lambda i: -f(data[i][K]))[:n_top]
for i in sorted(idx):
    d = data[i]
    top = sorted(stalls, key=lambda s: -f(d[s]))[:2]
    why = " ".join(f"{s[6:]}:{100*f(d[s])/max(f(d[K]),1):.0f}%" for s in top)
    print(f"{i:5d} {100*f(d[K])/tot:5.2f}% thr={d['Avg. Threads Executed']:>5} "
          f"{d['Source'].strip()[:64]:64s} {why}")
