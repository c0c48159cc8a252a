mkdir -p gpurun_out
CMD="python tools/run_pipeline.py --config ${CFG:-C3} --reps 2"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-gen_kernel} -s ${SKIP:-1} -c 1 -o gpurun_out/${OUT:-prof_gen} $CMD > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/prof_plain.log; tail -5 gpurun_out/ncu_full.log
