# A/B over VDI_WIDE_AFTER (narrow replays before the wide hand-off): gen time at
# C3 (N=1) and of one N=8 rank, plus generation parity.
mkdir -p gpurun_out
for wa in ${WAS:-99 3 2}; do
  VDI_NVCC_EXTRA="-DVDI_WIDE_AFTER=$wa" python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build fail"; continue; }
  echo "WIDE_AFTER $wa C3: $(timeout 300 python tools/run_pipeline.py --config C3 --reps 3 2>&1 | grep -o "'gen': [0-9.]*\|handed to the wide bisect [0-9]*" | tr '\n' ' ')"
  timeout 300 python tools/rank_gen_launches.py --world 8 > /dev/null 2>&1
  echo "  rank8 gen: $(timeout 300 python -c "
import sys,os; sys.path.insert(0,os.getcwd())
import torch
from paper_2206_08660_b200 import shard, synth
from paper_2206_08660_b200 import device as dv
from paper_2206_08660_b200.generate import GenParams
vol,tf,g,r,n=synth.config('C3')
p=shard.Pipeline(vol,tf,g,r,GenParams(n_sg=n),world=8,rank=0)
dv.launch_bricks(p.vol_dev,p.vt,p.res_dims,p.bricks)
ts=[]
for i in range(4):
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record(); p.generate_only(gather=False); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
print(ts)
" 2>&1 | tail -1)"
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
timeout 1200 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_full_c3.py 2>&1 | tail -3
