mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py -q --timeout 600 -x > gpurun_out/pytest_codec.log 2>&1; echo "pytest codec rc=$? $(tail -1 gpurun_out/pytest_codec.log)"
grep -E "Error|assert|FAIL|error" gpurun_out/pytest_codec.log | head -20
