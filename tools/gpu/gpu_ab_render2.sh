mkdir -p gpurun_out
for m in 1 5 6 8; do
  VDI_NVCC_EXTRA="-DVDI_RENDER_MINB=$m" python -m paper_2206_08660_b200.build > /dev/null 2>&1
  echo "MINB=$m"; timeout 300 python tools/run_pipeline.py --config C3 --reps 3 2>&1 | grep step | tail -2
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
