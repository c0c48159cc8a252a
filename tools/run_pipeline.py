"""Run generate (+ render) of a config a few times: the target command for ncu
captures (`ncu ... python tools/run_pipeline.py --config C3 --reps 2`)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2206_08660_b200 import shard, synth  # noqa: E402
from paper_2206_08660_b200.generate import GenParams  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C3")
p.add_argument("--reps", type=int, default=2)
p.add_argument("--no-ranges", action="store_true", help="render without VdiRenderArgs.list_range")
p.add_argument("--no-dyn", action="store_true", help="render without VdiRenderArgs.tile_counter")
a = p.parse_args()
from paper_2206_08660_b200.tuning import TUNING  # noqa: E402
if a.no_ranges:
    TUNING.list_ranges = False
if a.no_dyn:
    TUNING.dyn_tiles = False
vol, tf, gcam, rcam, n_sg = synth.config(a.config)
pipe = shard.Pipeline(vol, tf, gcam, rcam, GenParams(n_sg=n_sg))
for _ in range(a.reps):
    ev = pipe.step(timed=True)
    print({k: round(v, 3) for k, v in ev.items()}, flush=True)
torch.cuda.synchronize()
print("samples", pipe.samples_executed(), "render stats", pipe.exact_render_stats())
ctl = pipe.bufs.workspace[:512].view(torch.int64).cpu().tolist()
passes = pipe.bufs.passes.cpu()
hit = int((passes > 0).sum())
print(f"round0: queued rays {ctl[2]}, cached entries {ctl[1]} ({ctl[1]*16/1e9:.2f} GB), "
      f"deferred {ctl[4]}, handed to the wide bisect {ctl[7]}; hit rays {hit} of {passes.numel()}, "
      f"mean passes (hit) {float(passes[passes > 0].float().mean()):.2f}, "
      f"1-pass rays {int((passes == 1).sum())}")
# RoundCtl words 10..13: the VDI_BISECT_STATS counters, 14..16 VDI_FILL_STATS
if any(ctl[10:14]):
    print(f"bisect replays {ctl[13]}: visible steps {ctl[10]}, run steps {ctl[11]} "
          f"covering {ctl[12]} entries")
if any(ctl[14:17]):
    print(f"fill chunks {ctl[14]}: all in empty bricks {ctl[15]}, all transparent {ctl[16]}")
