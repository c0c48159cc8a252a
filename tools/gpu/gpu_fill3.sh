mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout 1400 > gpurun_out/pytest_fill.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_fill.log)"
for c in C3 C4 C5; do echo -n "$c "; timeout 600 python tools/run_pipeline.py --config $c --reps 3 2>&1 | grep step | tail -1; done
