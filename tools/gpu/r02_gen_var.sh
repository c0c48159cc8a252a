# Generation A/B over compile-time variants ($VARIANTS, ';'-separated, "" = default):
# C3 (+ $EXTRA_CFGS) gen times per variant, then the generation parity tests (+ $EXTRA_TESTS)
# on the default build.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "${VS[@]}"; do
  VDI_NVCC_EXTRA="$v" python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build '$v' failed"; continue; }
  for cfg in C3 ${EXTRA_CFGS}; do
    echo "[$v] $cfg: $(timeout 600 python tools/run_pipeline.py --config $cfg --reps 4 2>&1 | grep -o "'${KEY:-gen}': [0-9.]*" | tr '\n' ' ')"
  done
  [ -n "$TESTS_EACH" ] && timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py ${EXTRA_TESTS} 2>&1 | tail -1
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build failed"; exit 1; }
[ -z "$NO_TESTS" ] && timeout 1500 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_full_c3.py ${EXTRA_TESTS} 2>&1 | tail -3
