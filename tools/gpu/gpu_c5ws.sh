mkdir -p gpurun_out
for g in 24 64 120; do
  echo "WS=$g GB"; VDI_GEN_WS_GB=$g timeout 600 python tools/run_pipeline.py --config C5 --reps 2 2>&1 | grep -E "step|round0" | tail -2
done
