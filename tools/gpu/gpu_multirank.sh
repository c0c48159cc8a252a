mkdir -p gpurun_out
export VDI_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --e2e-steps 1 > gpurun_out/multirank2.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/multirank2.log | cut -c1-1500
