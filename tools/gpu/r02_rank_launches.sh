# ncu launch list (time only) of one rank's generation share (C3, N = 8, rank 0) + per-phase summary
mkdir -p gpurun_out
python -m paper_2206_08660_b200.build > /dev/null 2>&1 || exit 1
CMD="python tools/rank_gen_launches.py --config ${CFG:-C3} --world ${WORLD:-8} --rank 0"
timeout 600 $CMD > gpurun_out/rank_plain.log 2>&1 || { echo plain failed; tail gpurun_out/rank_plain.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,sm__warps_active.avg.per_cycle_active --clock-control none --csv --log-file gpurun_out/rank_launches.csv $CMD > gpurun_out/rank_ncu.log 2>&1; echo "ncu rc=$?"
