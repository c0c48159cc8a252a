mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bricked.py tests/test_gpu_parity.py tests/test_gpu_c5.py -q --timeout 1400 -x > gpurun_out/pytest_bricked.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_bricked.log)"
grep -E "Error|assert|FAIL|error" gpurun_out/pytest_bricked.log | head -20
timeout 300 python tools/run_pipeline.py --config C3 --reps 2 2>&1 | grep step | tail -1
