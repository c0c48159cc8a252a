mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/mc_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_blobs64 or stripes or random_vdis or search_fuzz or minimal" --timeout 1100 -p no:cacheprovider > gpurun_out/memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed|Invalid" gpurun_out/memcheck.log | head -10
