mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/smoke.log)"
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
grep -E "^FAILED|Error" gpurun_out/pytest_gpu.log | head
timeout 2000 python tools/config_table.py > gpurun_out/config_table.log 2>&1; echo "table rc=$?"; tail -8 gpurun_out/config_table.log
