# DVR round: GPU tests for DVR + timing at C2/C3/C4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dvr.py -q --timeout 600 > gpurun_out/pytest_dvr.log 2>&1; echo "pytest dvr rc=$? $(tail -1 gpurun_out/pytest_dvr.log)"
for c in C2 C3 C4; do timeout 600 python tools/bench_dvr.py --config $c --oracle-rows 4 >> gpurun_out/bench_dvr.log 2>&1; echo "$c rc=$?"; done
cat gpurun_out/bench_dvr.log | cut -c1-600
