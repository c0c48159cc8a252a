# Render with / without the per-list depth ranges (VdiRenderArgs.list_range) + render parity tests.
mkdir -p gpurun_out
python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
for cfg in ${CFGS:-C3 C4 C2}; do
  for flag in "" "--no-ranges"; do
    echo "$cfg $flag: $(timeout 300 python tools/run_pipeline.py --config $cfg --reps 4 $flag 2>&1 | grep -o "'render': [0-9.]*" | tr '\n' ' ')"
  done
done
timeout 1200 python -m pytest -q -x tests/test_gpu_tiles.py tests/test_gpu_parity.py tests/test_gpu_full_c3.py tests/test_gpu_rshaped.py tests/test_gpu_acceptance.py 2>&1 | tail -3
