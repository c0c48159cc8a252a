mkdir -p gpurun_out
python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build failed"; exit 1; }
timeout 1500 python -m pytest -q -x tests/test_gpu_exchange.py tests/test_gpu_stream.py tests/test_gpu_shard.py tests/test_gpu_bricked.py tests/test_gpu_multirank_bench.py 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 4 --cpu-seconds 6 > gpurun_out/r02_bench_try.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/r02_bench_try.log
timeout 1200 python tools/rank_shares.py --config C3 --worlds 1,2,4,8 > gpurun_out/r02_rank_shares_c3.log 2>&1; echo "rs rc=$?"; tail -8 gpurun_out/r02_rank_shares_c3.log
