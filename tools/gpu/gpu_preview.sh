mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_preview.py -q --timeout 600 -x > gpurun_out/pytest_preview.log 2>&1; echo "pytest preview rc=$? $(tail -1 gpurun_out/pytest_preview.log)"
tail -30 gpurun_out/pytest_preview.log | grep -E "Error|assert|FAIL" | head -20
timeout 600 python tools/bench_preview.py --config C2 --oracle > gpurun_out/bench_preview.log 2>&1; echo "C2 rc=$?"
timeout 600 python tools/bench_preview.py --config C3 >> gpurun_out/bench_preview.log 2>&1; echo "C3 rc=$?"
cut -c1-400 gpurun_out/bench_preview.log
