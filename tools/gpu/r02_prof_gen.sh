mkdir -p gpurun_out
CMD="python tools/run_pipeline.py --config C3 --reps 1"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gen_(bisect|fill|sample|emit)" -c 4 -o gpurun_out/r02_gen_phases $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu_full.log
