# Per compile-time variant ($VARIANTS, ';'-separated): C3 gen (N = 1) and the C3 N = 8
# rank-share projection (tools/rank_shares.py --worlds 8), then (TESTS=1) generation parity.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "${VS[@]}"; do
  VDI_NVCC_EXTRA="$v" python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build '$v' failed"; continue; }
  echo "[$v] C3 N=1: $(timeout 600 python tools/run_pipeline.py --config C3 --reps 4 2>&1 | grep -o "'gen': [0-9.]*" | tr '\n' ' ')"
  echo "[$v] C3 N=8: $(timeout 900 python tools/rank_shares.py --config C3 --worlds ${WORLDS:-8} --reps 2 2>&1 | grep '^{' | python -c "import sys,json; [print('world', d['world'], 'slowest', round(d['kernels_ms_max'],2), 'gen', [round(r['gen'],2) for r in d['ranks']]) for d in map(json.loads, sys.stdin)]")"
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
[ -n "$TESTS" ] && timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_full_c3.py tests/test_gpu_bricked.py 2>&1 | tail -2
