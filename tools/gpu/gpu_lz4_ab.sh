# LZ4 A/B: codec parity tests (both table sizes), bench_codec per table size, launch list
mkdir -p gpurun_out
for hl in 13 12 11; do
VDI_LZ4_HASHLOG=$hl timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_acceptance.py -q --timeout 600 -x > gpurun_out/pytest_codec.log 2>&1; echo "hl=$hl pytest codec rc=$? $(tail -1 gpurun_out/pytest_codec.log)"
grep -E "Error|assert|FAIL" gpurun_out/pytest_codec.log | head -10
done
for hl in 13 12 11; do
  VDI_LZ4_HASHLOG=$hl timeout 600 python tools/bench_codec.py --config C3 --reps 5 2>&1 | tail -1 | cut -c1-330
done
VDI_LZ4_HASHLOG=12 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lz4" --csv \
  --log-file gpurun_out/lz4_launches.csv python tools/bench_codec.py --config C3 --reps 1 > /dev/null 2>&1; echo "launch rc=$?"
grep gpu__time gpurun_out/lz4_launches.csv | head -6 | awk -F'","' '{print $5, $NF}' | cut -c1-30,100-
