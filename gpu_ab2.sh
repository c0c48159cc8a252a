for v in $VARIANTS; do
  export VDI_BISECT_VARIANT=$v
  r=$(timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "generate" --timeout 250 2>&1 | tail -1)
  t=$(timeout 300 python tools/run_pipeline.py --config C3 --reps 3 2>&1 | grep step | tail -1)
  echo "$v | $r | $t"
done
