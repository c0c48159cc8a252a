# full measurement round: tests, bench, launch list with DRAM metrics
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
bash gpu_launch.sh > gpurun_out/launch_summary.txt 2>&1; echo "launch rc=$?"
tail -1 gpurun_out/bench_full.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ['value','ms_per_step','phases_ms']}, d['roofline']['frac'], d['e2e'], d.get('cpu_baseline'))"
