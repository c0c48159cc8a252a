# VDI1 unpack: codec / exchange tests (TESTS=1) and one N = 8 C3 rank's decode time
python -m paper_2206_08660_b200.build >/dev/null 2>&1 || exit 1
[ -n "$TESTS" ] && timeout 900 python -m pytest -q -x tests/test_gpu_codec.py tests/test_gpu_exchange.py tests/test_gpu_shard.py 2>&1 | tail -1
timeout 900 python tools/rank_shares.py --config C3 --worlds 8 --reps 3 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('decode ms per rank', [round(r['decode'],3) for r in d['ranks']], 'slowest', round(d['kernels_ms_max'],2), 'proj', round(d['projected_speedup'],2))"
