# LZ4 kernels: plain timing, per-kernel launch list, one ncu --set full of the parse kernel
mkdir -p gpurun_out
C="python tools/bench_codec.py --config C3 --reps 3"
$C > gpurun_out/lz4_plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/lz4_plain.log | cut -c1-400
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"lz4|enc_" --csv \
  --log-file gpurun_out/lz4_launches.csv $C > /dev/null 2>&1; echo "launch rc=$?"
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/lz4_launches.csv")) if len(r) > 14 and r[0].isdigit()]
agg = {}
for r in rows:
    agg.setdefault((int(r[0]), r[4][:40]), {})[r[12]] = r[14]
for (i, k), m in sorted(agg.items())[:24]:
    print(i, k, m)
PY
ncu --set full --clock-control none --import-source on -k regex:lz4_parse -c 1 -o gpurun_out/prof_lz4 $C > gpurun_out/ncu_lz4.log 2>&1; echo "full rc=$?"
