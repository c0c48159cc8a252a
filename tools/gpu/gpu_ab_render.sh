# render A/B over VDI_RENDER_MINB: render parity tests + C3 / C4 timing per value
mkdir -p gpurun_out
for m in ${1:-5 6}; do
  VDI_NVCC_EXTRA="-DVDI_RENDER_MINB=$m" python -m paper_2206_08660_b200.build > /dev/null 2>&1
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "render or c4" --timeout 800 > gpurun_out/ab_render_$m.log 2>&1
  echo "MINB=$m tests: $(tail -1 gpurun_out/ab_render_$m.log)"
  for c in C3 C4; do echo -n "$c "; timeout 300 python tools/run_pipeline.py --config $c --reps 3 2>&1 | grep step | tail -1; done
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
