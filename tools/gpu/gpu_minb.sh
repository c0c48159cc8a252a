# A/B over a launch-bounds macro: bash gpu_minb.sh MACRO "v1 v2 ..." (rebuilds per value)
mkdir -p gpurun_out
for v in $2; do
  VDI_NVCC_EXTRA="-D$1=$v" python -m paper_2206_08660_b200.build -v > gpurun_out/build_$v.log 2>&1 || { echo "build $v failed"; tail -5 gpurun_out/build_$v.log; continue; }
  grep -A1 "gen_fill_kernelILi16" gpurun_out/build_$v.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | head -2 | tr '\n' ' '
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "generate" --timeout 500 > gpurun_out/ab_$v.log 2>&1
  echo "$1=$v tests: $(tail -1 gpurun_out/ab_$v.log)"
  for c in ${CFGS:-C3}; do echo "$c $(timeout 600 python tools/run_pipeline.py --config $c --reps 3 2>&1 | grep step | tail -1)"; done
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
