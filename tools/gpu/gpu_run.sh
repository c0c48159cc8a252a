# usage: bash gpu_run.sh [bench args...]
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -rA --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/smoke.log; grep -E "PASSED|FAILED|ERROR|passed|failed" gpurun_out/pytest_gpu.log | tail -30; tail -2 gpurun_out/bench.log
