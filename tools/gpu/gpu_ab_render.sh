# stream packed e2e + render A/B over register budgets
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_parity.py -q --timeout 600 -x -k "stream or render" > gpurun_out/pytest_sr.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_sr.log)"
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 6 --no-cpu-baseline > gpurun_out/bench_short.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_short.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e']['value'],'dense',d['e2e']['dense']['value'],'render ms',d['phases_ms']['render'])"
for m in 1 5 6; do
  VDI_NVCC_EXTRA="-DVDI_RENDER_MINB=$m" python -m paper_2206_08660_b200.build > /dev/null 2>&1
  echo "MINB=$m"; timeout 300 python tools/run_pipeline.py --config C3 --reps 3 2>&1 | grep step | tail -2
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
