# run_pipeline.py render / gen times per flag set ($FLAGSETS, ';'-separated) and config,
# then (TESTS=1) the render parity tests.
mkdir -p gpurun_out
python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
IFS=';' read -ra FS <<< "${FLAGSETS:-;--no-dyn}"
for cfg in ${CFGS:-C3 C4 C2}; do
  for f in "${FS[@]}"; do
    echo "$cfg [$f]: $(timeout 300 python tools/run_pipeline.py --config $cfg --reps 4 $f 2>&1 | grep -o "'${KEY:-render}': [0-9.]*" | tr '\n' ' ')"
  done
done
[ -n "$TESTS" ] && timeout 1200 python -m pytest -q -x tests/test_gpu_tiles.py tests/test_gpu_parity.py tests/test_gpu_full_c3.py tests/test_gpu_rshaped.py 2>&1 | tail -3
if [ -n "$PROF" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 -o gpurun_out/$PROF python tools/run_pipeline.py --config C3 --reps 2 > gpurun_out/ncu_flags.log 2>&1; echo "ncu rc=$?"
fi
