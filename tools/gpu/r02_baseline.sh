# Round-2 baseline evidence: render ncu --set full (source page) at C3, and a
# per-kernel metric list (time, DRAM bytes, FP64 pipe, warp efficiency, L2 hit)
# for one C3 and one C5 pipeline step.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__thread_inst_executed_per_inst_executed.ratio,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
CMD="python tools/run_pipeline.py --config C3 --reps 2"
$CMD > gpurun_out/r02_plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 -o gpurun_out/r02_render $CMD > gpurun_out/r02_ncu_render.log 2>&1
echo "render rc=$?"
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_c3_metrics.csv $CMD > gpurun_out/r02_ncu_c3m.log 2>&1
echo "c3 metrics rc=$?"
CMD5="python tools/run_pipeline.py --config C5 --reps 1"
$CMD5 > gpurun_out/r02_plain_c5.log 2>&1 && \
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_c5_metrics.csv $CMD5 > gpurun_out/r02_ncu_c5m.log 2>&1
echo "c5 metrics rc=$?"
tail -3 gpurun_out/r02_plain_c3.log gpurun_out/r02_plain_c5.log
