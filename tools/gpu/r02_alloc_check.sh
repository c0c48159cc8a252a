python -m paper_2206_08660_b200.build > /dev/null 2>&1 || exit 1
for cfg in C3 C4; do echo "$cfg: $(timeout 600 python tools/run_pipeline.py --config $cfg --reps 4 2>&1 | grep -o "'gen': [0-9.]*" | tr '\n' ' ')"; done
timeout 600 python tools/run_pipeline.py --config C3 --reps 2 2>&1 | tail -2
timeout 2000 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_full_c3.py tests/test_gpu_full_c4.py tests/test_gpu_c5.py tests/test_gpu_bricked.py tests/test_gpu_stream.py tests/test_gpu_rshaped.py 2>&1 | tail -2
timeout 900 python tools/rank_shares.py --config C3 --worlds 1,8 --reps 2 2>&1 | tail -5
