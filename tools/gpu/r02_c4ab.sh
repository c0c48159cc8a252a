# C3 / C4 generation per compile-time variant ($VARIANTS, ';'-separated), then (TESTS=1) generation parity
IFS=';' read -ra VS <<< "${VARIANTS:- }"
for v in "${VS[@]}"; do
  VDI_NVCC_EXTRA="$v" python -m paper_2206_08660_b200.build > /dev/null 2>&1
  for cfg in ${CFGS:-C3 C4}; do
    echo "[$v] $cfg: $(timeout 600 python tools/run_pipeline.py --config $cfg --reps 3 2>&1 | grep -o "'gen': [0-9.]*" | tr '\n' ' ')"
  done
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
[ -n "$TESTS" ] && timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_full_c3.py tests/test_gpu_full_c4.py tests/test_gpu_bricked.py tests/test_gpu_c5.py 2>&1 | tail -1
true
