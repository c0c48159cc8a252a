mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_singles.py -q --timeout 800 > gpurun_out/pytest_singles.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_singles.log)"
grep -E "^FAILED|Error|assert" gpurun_out/pytest_singles.log | head -20
