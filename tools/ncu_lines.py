"""Per-CUDA-source-line instruction counts and stall samples of an ncu report
(ncu -i X --page source --csv --print-source=cuda,sass). usage:
python tools/ncu_lines.py X.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv",
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(io.StringIO(out)))
fname, data = None, []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9 or r[2] != "-":
        continue  # only the CUDA-line aggregate rows (Address "-")
    try:
        data.append((float(r[7] or 0), float(r[4] or 0), float(r[10] or 0), fname, r[0],
                     r[1].strip()))
    except ValueError:
        pass
ti = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for d in sorted(data, key=lambda x: -x[0])[:n_top]:
    print(f"{100 * d[0] / ti:5.1f}% inst {100 * d[1] / ts:5.1f}% smp thr={d[2]:4.1f} "
          f"{d[3]}:{d[4]:<5} {d[5][:90]}")
