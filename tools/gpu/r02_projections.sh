# Rank-share projections (tools/rank_shares.py) at HEAD: C3 interleaved N = 1, 2, 4, 8;
# C5 replicated and C5 bricked with balanced bands, N = 1, 8. Logs to gpurun_out/r02_rs_*.log.
mkdir -p gpurun_out
python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build failed"; exit 1; }
timeout 1200 python tools/rank_shares.py --config C3 --worlds 1,2,4,8 > gpurun_out/r02_rs_c3.log 2>&1; echo "c3 rc=$?"; tail -6 gpurun_out/r02_rs_c3.log
timeout 1800 python tools/rank_shares.py --config C5 --worlds 1,8 --reps 2 > gpurun_out/r02_rs_c5.log 2>&1; echo "c5 rc=$?"; tail -4 gpurun_out/r02_rs_c5.log
timeout 1800 python tools/rank_shares.py --config C5 --worlds 1,8 --reps 2 --bricked --balanced > gpurun_out/r02_rs_c5_bricked_balanced.log 2>&1; echo "c5b rc=$?"; tail -4 gpurun_out/r02_rs_c5_bricked_balanced.log
