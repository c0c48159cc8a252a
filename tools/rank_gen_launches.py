"""One rank's generation of an N-rank split (no collectives), twice: the
target of an ncu launch list (per-phase times of a rank's share).

    python tools/rank_gen_launches.py --config C3 --world 8 --rank 0"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2206_08660_b200 import shard, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200.generate import GenParams  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--world", type=int, default=8)
p.add_argument("--rank", type=int, default=0)
a = p.parse_args()
vol, tf, gcam, rcam, n_sg = synth.config(a.config)
pipe = shard.Pipeline(vol, tf, gcam, rcam, GenParams(n_sg=n_sg), world=a.world, rank=a.rank)
if pipe.slabs is not None:
    dv.launch_bricks(pipe.vol_dev, pipe.vt, pipe.res_dims, pipe.bricks)
for _ in range(2):
    pipe.generate_only(gather=False)
torch.cuda.synchronize()
print("ok", pipe.samples_executed())
