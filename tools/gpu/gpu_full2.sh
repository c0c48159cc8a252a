mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'prep',d['phases_ms']['prep'],'e2e',d['e2e']['value'],'dense',d['e2e']['dense']['value'],'serial',d['e2e']['serial']['value'],'render',d['phases_ms']['render'])"
