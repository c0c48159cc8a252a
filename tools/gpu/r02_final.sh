# Round-2 final evidence: GPU tests + smoke, the default bench line, the bench's ncu launch
# list, per-kernel metrics of one C3 step, ncu --set full of the generation phases and the
# render, the C1-C5 config table and the rank-share projections.
mkdir -p gpurun_out
bash tools/gpu/r02_evidence.sh
timeout 2400 python tools/config_table.py > gpurun_out/r02_config_table.log 2>&1; echo "config table rc=$?"
bash tools/gpu/r02_projections.sh
