mkdir -p gpurun_out
CMD="python tools/run_pipeline.py --config C3 --reps 2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'gen_(sample|fill)' -s 6 -c 2 -o gpurun_out/prof_sf $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
