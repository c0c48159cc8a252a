mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_dvr.py -q -x --timeout 1100 > gpurun_out/pytest_cz.log 2>&1; echo "tests: $(tail -1 gpurun_out/pytest_cz.log)"
grep -E "^FAILED|Error|assert" gpurun_out/pytest_cz.log | head
for z in 0 1; do export VDI_CELLS_Z=$z; echo "CELLS_Z=$z"; for c in C3 C5; do echo -n "$c "; timeout 600 python tools/run_pipeline.py --config $c --reps 3 2>&1 | grep step | tail -1; done; timeout 300 python tools/bench_dvr.py --config C3 | cut -c1-140; done
