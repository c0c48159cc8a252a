mkdir -p gpurun_out
CMD="python tools/run_pipeline.py --config C3 --reps 2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 -o gpurun_out/${OUT:-r02_render_v2} $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu_full.log
