# Render A/B over a compile-time variant: VAR="-DX=1 ..." values in $VARIANTS ("" = default),
# C3 / C4 render times, then the render parity tests on the last variant, and an ncu
# capture of the default render.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-;-DVDI_RANGE_AHEAD=1}"
for v in "${VS[@]}"; do
  VDI_NVCC_EXTRA="$v" python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build '$v' failed"; continue; }
  for cfg in ${CFGS:-C3 C4}; do
    echo "[$v] $cfg: $(timeout 300 python tools/run_pipeline.py --config $cfg --reps 4 2>&1 | grep -o "'render': [0-9.]*" | tr '\n' ' ')"
  done
  [ -n "$TESTS" ] && timeout 900 python -m pytest -q -x tests/test_gpu_tiles.py tests/test_gpu_parity.py tests/test_gpu_full_c3.py 2>&1 | tail -1
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
if [ -n "$PROF" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 -o gpurun_out/$PROF python tools/run_pipeline.py --config C3 --reps 2 > gpurun_out/ncu_render_var.log 2>&1; echo "ncu rc=$?"
fi
