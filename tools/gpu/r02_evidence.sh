# Round-2 evidence pass at HEAD: build, GPU tests, smoke, the default bench line,
# the bench's ncu launch list, the per-kernel metrics of one C3 step, and
# ncu --set full captures of the generation phases and the render.
#   gpurun --timeout 4200 -- 'bash tools/gpu/r02_evidence.sh'
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build.log 2>&1 || { echo build failed; tail gpurun_out/r02_build.log; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -v "^$" > gpurun_out/r02_gputests.log; echo "pytest rc=${PIPESTATUS[0]}"; tail -3 gpurun_out/r02_gputests.log
  python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02_smoke.log
fi
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02_bench.log | cut -c1-400
BCMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $BCMD > gpurun_out/r02_bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_bench_launches.csv $BCMD > gpurun_out/r02_ncu_bench.log 2>&1
echo "bench launch list rc=$?"
PCMD="python tools/run_pipeline.py --config C3 --reps 2"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__thread_inst_executed_per_inst_executed.ratio,lts__t_sector_hit_rate.pct
timeout 600 $PCMD > gpurun_out/r02_pipe_plain.log 2>&1 && \
timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_c3_metrics.csv $PCMD > gpurun_out/r02_ncu_metrics.log 2>&1
echo "metrics rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gen_(bisect|fill|sample|emit)" -c 4 -o gpurun_out/r02_gen_phases $PCMD > gpurun_out/r02_ncu_gen.log 2>&1
echo "gen full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 1 -c 1 -o gpurun_out/r02_render $PCMD > gpurun_out/r02_ncu_render.log 2>&1
echo "render full rc=$?"
