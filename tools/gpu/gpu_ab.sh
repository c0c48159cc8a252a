# A/B runs: bash gpu_ab.sh VAR "v1 v2 ..."  (runs gen parity tests + C3 pipeline per value)
mkdir -p gpurun_out
for v in $2; do
  export $1=$v
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "generate" --timeout 500 > gpurun_out/ab_$v.log 2>&1
  echo "$1=$v tests: $(tail -1 gpurun_out/ab_$v.log)"
  timeout 300 python tools/run_pipeline.py --config C3 --reps 3 2>&1 | grep step | tail -1
done
