mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_c5.py -q -x --timeout 1400 > gpurun_out/pytest_ns.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_ns.log)"
grep -E "^FAILED|Error|assert" gpurun_out/pytest_ns.log | head
for c in C2 C3 C4 C5; do echo -n "$c "; timeout 600 python tools/run_pipeline.py --config $c --reps 3 2>&1 | grep step | tail -1; done
