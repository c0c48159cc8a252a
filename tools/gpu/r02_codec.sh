mkdir -p gpurun_out
python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build failed"; exit 1; }
timeout 900 python -m pytest -q -x tests/test_gpu_codec.py tests/test_gpu_acceptance.py 2>&1 | tail -4
timeout 600 python tools/bench_codec.py --config C3 --reps 5 --cpu 2>&1 | tail -1 | tee gpurun_out/r02_bench_codec.jsonl
