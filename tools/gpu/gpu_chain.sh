mkdir -p gpurun_out
for v in 0 4 6; do
  export VDI_CHAIN_LEVELS=$v
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout 800 > gpurun_out/chain_$v.log 2>&1
  echo "CHAIN=$v tests: $(tail -1 gpurun_out/chain_$v.log)"
  for c in C3 C4 C5; do echo -n "$c "; timeout 600 python tools/run_pipeline.py --config $c --reps 2 2>&1 | grep step | tail -1; done
done
