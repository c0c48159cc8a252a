# A/B of the learned chain directions (VDI_LEARN_CHAIN): generation parity + timings
mkdir -p gpurun_out
for v in 0 1; do
  export VDI_LEARN_CHAIN=$v
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout 800 > gpurun_out/learn_$v.log 2>&1
  echo "LEARN=$v tests: $(tail -1 gpurun_out/learn_$v.log)"
  for c in C2 C3 C4 C5; do echo -n "$c "; timeout 600 python tools/run_pipeline.py --config $c --reps 3 2>&1 | grep step | tail -1; done
done
