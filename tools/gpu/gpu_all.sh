# everything the round end checks, plus the per-config table and the bench line
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/smoke.log)"
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head
timeout 1500 python tools/config_table.py --cpu-rows 4 > gpurun_out/config_table.log 2>&1; echo "table rc=$?"; tail -7 gpurun_out/config_table.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e']['value'],'dense',d['e2e']['dense']['value'],'serial',d['e2e']['serial']['value'],'frac',d['roofline']['frac'],d['phases_ms'])"
for c in C3 C4; do timeout 600 python tools/bench_dvr.py --config $c --oracle-rows 16 >> gpurun_out/bench_dvr.log 2>&1; done
timeout 900 python tools/bench_preview.py --config C3 > gpurun_out/bench_preview.log 2>&1
timeout 900 python tools/bench_preview.py --config C2 --oracle >> gpurun_out/bench_preview.log 2>&1
timeout 600 python tools/bench_codec.py --config C3 --cpu > gpurun_out/bench_codec.log 2>&1
echo "done"
