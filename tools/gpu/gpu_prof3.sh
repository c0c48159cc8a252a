mkdir -p gpurun_out
CMD="python tools/run_pipeline.py --config ${CFG:-C3} --reps 2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-3} -c 1 -o gpurun_out/${OUT} $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_full.log
