mkdir -p gpurun_out
CMD="python tools/run_pipeline.py --config ${CFG:-C3} --reps 2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'gen_(sample|bisect)' -s 6 -c 2 -o gpurun_out/${OUT:-prof_gen2} $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu_full.log
