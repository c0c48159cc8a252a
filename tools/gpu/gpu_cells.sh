# corner-record build: parity tests that use cells, pipeline timing, kernel times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_bricked.py -q --timeout 800 -x > gpurun_out/pytest_cells.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_cells.log)"
grep -E "^FAILED|Error" gpurun_out/pytest_cells.log | head -5
for c in C3 C5; do timeout 600 python tools/run_pipeline.py --config $c --reps 3 2>&1 | grep step | tail -1; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"cells|brick_max" --csv \
  --log-file gpurun_out/cells_launches.csv python tools/run_pipeline.py --config C3 --reps 1 > /dev/null 2>&1; echo "launch rc=$?"
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/cells_launches.csv")) if len(r) > 14 and r[0].isdigit()]
agg = {}
for r in rows:
    agg.setdefault((int(r[0]), r[4][:30]), {})[r[12].split("__")[1][:12]] = r[14]
for (i, k), m in sorted(agg.items())[:6]:
    print(i, k, m)
PY
