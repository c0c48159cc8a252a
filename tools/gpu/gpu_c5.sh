mkdir -p gpurun_out
free -g | head -2; nproc
timeout 600 python tools/run_pipeline.py --config C5 --reps 2 > gpurun_out/c5_pipeline.log 2>&1; echo "pipeline rc=$?"; tail -4 gpurun_out/c5_pipeline.log
timeout 1200 python -m pytest tests/test_gpu_c5.py -q --timeout 1100 -x > gpurun_out/pytest_c5.log 2>&1; echo "pytest c5 rc=$? $(tail -1 gpurun_out/pytest_c5.log)"
grep -E "Error|assert|FAIL|error|SKIP" gpurun_out/pytest_c5.log | head -20
