for spec in ${SPECS}; do
  VDI_NVCC_EXTRA="$(echo $spec | tr ',' ' ')" python -m paper_2206_08660_b200.build > /dev/null 2>&1 || { echo "build fail $spec"; continue; }
  echo "$spec C3: $(timeout 300 python tools/run_pipeline.py --config C3 --reps 3 2>&1 | grep -o "'gen': [0-9.]*\|handed to the wide bisect [0-9]*" | tr '\n' ' ')"
  echo "   rank8: $(timeout 300 python -c "
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
    a.record(); p.generate_only(gather=False); b.record(); b.synchronize(); ts.append(round(a.elapsed_time(b),2))
print(ts)
" 2>&1 | tail -1)"
done
python -m paper_2206_08660_b200.build > /dev/null 2>&1
