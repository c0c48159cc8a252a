# Full evidence pass: GPU tests, smoke, the default bench line.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02_build.log 2>&1 || { echo build failed; tail gpurun_out/r02_build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -v "^$" > gpurun_out/r02_gputests.log; echo "pytest rc=${PIPESTATUS[0]}"; tail -3 gpurun_out/r02_gputests.log; grep PARITY gpurun_out/r02_gputests.log | cut -c1-300
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/r02_bench.log
