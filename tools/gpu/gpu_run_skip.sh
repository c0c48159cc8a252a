mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_dvr.py tests/test_gpu_c5.py tests/test_gpu_bricked.py -q -x --timeout 1400 > gpurun_out/pytest_skip.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_skip.log)"
grep -E "^FAILED|Error|assert" gpurun_out/pytest_skip.log | head
for c in C3 C4 C5; do echo -n "$c "; timeout 600 python tools/run_pipeline.py --config $c --reps 2 2>&1 | grep step | tail -1; done
timeout 600 python tools/bench_dvr.py --config C3 | cut -c1-200
