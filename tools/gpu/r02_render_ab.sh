# Render A/B over the launch bound (VDI_RENDER_MINB) + render parity tests.
mkdir -p gpurun_out
for mb in ${MBS:-6 5 4}; do
  VDI_NVCC_EXTRA="-DVDI_RENDER_MINB=$mb" python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build $mb failed"; continue; }
  for cfg in C3 C4; do
    echo "MINB $mb $cfg: $(timeout 300 python tools/run_pipeline.py --config $cfg --reps 3 2>&1 | grep -o "'render': [0-9.]*" | tr '\n' ' ')"
  done
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_singles.py tests/test_gpu_acceptance.py 2>&1 | tail -5
