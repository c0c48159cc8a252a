# full measurement round: smoke, tests, bench, launch lists (bench + pipeline with DRAM metrics)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
BCMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $BCMD > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv $BCMD > gpurun_out/ncu_bench.log 2>&1
echo "bench launch list rc=$?"
bash tools/gpu/gpu_launch.sh > gpurun_out/launch_summary.txt 2>&1; echo "launch rc=$?"
python tools/summarize_launches.py gpurun_out/launches.csv gpurun_out/c3_gen_traffic.json "ncu launch list of tools/run_pipeline.py --config C3 --reps 2"
tail -1 gpurun_out/bench_full.log | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ['value','ms_per_step','phases_ms']}, d['roofline']['frac'], d['e2e'], d.get('cpu_baseline'))"
