mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_acceptance.py tests/test_gpu_stream.py -q --timeout 600 -x > gpurun_out/pytest_codec.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_codec.log)"
timeout 600 python tools/bench_codec.py --config C3 --reps 5 --cpu > gpurun_out/bench_codec.log 2>&1; tail -1 gpurun_out/bench_codec.log | cut -c1-600
