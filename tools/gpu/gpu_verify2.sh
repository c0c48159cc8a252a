mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py -q --timeout 600 -x > gpurun_out/pytest_stream.log 2>&1; echo "pytest stream rc=$? $(tail -1 gpurun_out/pytest_stream.log)"
grep -E "Error|assert|FAIL" gpurun_out/pytest_stream.log | head
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['e2e']['d2h_bytes_per_step'], d['e2e']['dense']['value'], d['e2e']['serial']['value'], d['roofline']['frac'])"
