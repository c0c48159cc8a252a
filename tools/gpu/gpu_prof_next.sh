# ncu --set full captures of the SURVEY 8(f) kernels (each after a plain run of the same command)
mkdir -p gpurun_out
C1="python tools/bench_dvr.py --config C3 --reps 1"
$C1 > gpurun_out/p_dvr_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dvr_kernel -c 1 -o gpurun_out/prof_dvr $C1 > gpurun_out/ncu_dvr.log 2>&1; echo "dvr rc=$?"
C2="python tools/bench_preview.py --config C2 --reps 1"
$C2 > gpurun_out/p_prev_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:preview_warp -c 1 -o gpurun_out/prof_preview $C2 > gpurun_out/ncu_prev.log 2>&1; echo "preview rc=$?"
C3="python tools/bench_codec.py --config C3 --reps 1"
$C3 > gpurun_out/p_codec_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"lz4_parse|enc_segs" -c 2 -o gpurun_out/prof_codec $C3 > gpurun_out/ncu_codec.log 2>&1; echo "codec rc=$?"
