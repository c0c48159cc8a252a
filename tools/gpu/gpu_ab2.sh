# A/B of VDI_BISECT_VARIANT values: gen parity subset, C3 step timing, and
# (PHASES=1) per-kernel times from an ncu launch list
for v in $VARIANTS; do
  export VDI_BISECT_VARIANT=$v
  r=$(timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "generate" --timeout 250 2>&1 | tail -1)
  t=$(timeout 300 python tools/run_pipeline.py --config C3 --reps 3 2>&1 | grep step | tail -1)
  echo "$v | $r | $t"
  if [ -n "$PHASES" ]; then
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ph.csv \
      python tools/run_pipeline.py --config C3 --reps 1 > /dev/null 2>&1
    echo "   $(python tools/phase_times.py gpurun_out/ph.csv)"
  fi
done
