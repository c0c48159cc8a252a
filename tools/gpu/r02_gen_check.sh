# Generation change check: C3 phase timings (+C4/C5 when FULL=1) and the
# generation parity tests (golden fixtures, minimal workspace, full-frame C3).
mkdir -p gpurun_out
python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build failed"; exit 1; }
for cfg in C3 ${EXTRA_CFGS}; do
  echo "$cfg: $(timeout 600 python tools/run_pipeline.py --config $cfg --reps 3 2>&1 | grep -o "'gen': [0-9.]*" | tr '\n' ' ')"
done
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_full_c3.py ${EXTRA_TESTS} 2>&1 | tail -4
