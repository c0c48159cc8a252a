"""Per-rank work of an N-GPU run, timed on ONE GPU (VERDICT r1
"multi-GPU readiness without an 8-GPU node").

For N = 1, 2, 4, 8 every rank's share of a step runs here, one rank after
another (no rank waits on another): its slab of the brick maxima, its
generation rows (+ partial AccelGrid), its VDI1 packing for the exchange, the
unpacking of all N shards, and its output rows of the render (over the full
VDI). The collectives are not run -- one GPU cannot stand in for NVLink --
but modelled from their byte counts at the measured NVLink figures of
B200_PROFILING.md (8-rank all-reduce bus bandwidth 725 GB/s, all-gather at
the same rate, + 20 us launch latency per collective). A step at N is the
slowest rank's kernels + the collectives; the projection is t(1) / t(N).

    python tools/rank_shares.py --config C3 [--worlds 1,2,4,8] [--reps 3]
    python tools/rank_shares.py --config C5 --bricked --worlds 1,8

--bricked: contiguous generation bands, each rank keeping only its voxel box
resident (shard.band_volume_box), the C5 placement; the render keeps the
interleaved bands.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2206_08660_b200 import _capi, shard, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from paper_2206_08660_b200 import generate as gen  # noqa: E402
from paper_2206_08660_b200.generate import GenParams, launch_generate  # noqa: E402
from paper_2206_08660_b200.raycast import alloc_zmask, launch_zmask, render_args  # noqa: E402
from paper_2206_08660_b200.vdi import DeviceVdi  # noqa: E402

BUS_GBPS = 725.0  # B200_PROFILING.md: 8-rank all-reduce bus bandwidth at 1 GiB
LAT_US = 20.0     # per collective


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed(fn, reps):
    fn()  # warm-up: first-call allocations (workspace, caches) are not timed
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def coll_ms(nbytes, world, kind):
    if world <= 1:
        return 0.0
    f = 2.0 * (world - 1) / world if kind == "allreduce" else (world - 1) / world
    return f * nbytes / (BUS_GBPS * 1e9) * 1e3 + LAT_US / 1e3


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C3")
    p.add_argument("--worlds", default="1,2,4,8")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--bricked", action="store_true")
    p.add_argument("--balanced", action="store_true",
                   help="bricked bands of unequal height balanced on the per-row executed "
                        "samples of the N = 1 step (as the previous frame would give them)")
    p.add_argument("--cells-max-world", type=int, default=None,
                   help="tuning.TUNING.cells_max_world (corner records on ranks up to this N)")
    a = p.parse_args()
    if a.cells_max_world is not None:
        from paper_2206_08660_b200.tuning import TUNING
        TUNING.cells_max_world = a.cells_max_world
    vol, tf, gcam, rcam, n_sg = synth.config(a.config)
    params = GenParams(n_sg=n_sg)
    L = _capi.load()
    box_volume = None
    if a.config == "C5":
        box_volume = lambda org, size: synth.rm_like(box=(org, size)).device_data  # noqa: E731
    # the full VDI every rank's render reads after the exchange
    ref = shard.Pipeline(vol, tf, gcam, rcam, params)
    ref.step()
    torch.cuda.synchronize()
    full_vdi = DeviceVdi(ref.bufs.counts, ref.bufs.segs, sorted=True)
    row_cost = ref.bufs.samples.sum(dim=1).double().cpu().numpy()
    ref.bufs.workspace = None  # the ranks below size their own generation scratch
    torch.cuda.empty_cache()
    ref_grid = ref.bufs.grid
    w, h = gcam.viewport
    ow, oh = rcam.viewport
    rows_out = []
    base_step = None
    for world in [int(x) for x in a.worlds.split(",")]:
        ranks = []
        for r in range(world):
            gen.release_workspace()
            torch.cuda.empty_cache()
            bounds = (shard.balance_bands(row_cost, world)
                      if a.bricked and a.balanced and world > 1 else None)
            pipe = shard.Pipeline(vol, tf, gcam, rcam, params, world=world, rank=r,
                                  bricked=a.bricked and world > 1, box_volume=box_volume,
                                  band_bounds=bounds)
            if pipe.slabs is not None:  # the other ranks' slabs, as the all-gather leaves them
                dv.launch_bricks(pipe.vol_dev, pipe.vt, pipe.res_dims, pipe.bricks)
            prep_ms = timed(lambda: pipe.prep(pipe.vol_dev, gather=False), a.reps)

            def run_gen():
                launch_generate(pipe.vol_dev, pipe.vt, pipe.vol.dims, pipe.lut_dev, pipe.gcam,
                                pipe.aabb, pipe.params, pipe.resolved, pipe.bufs, pipe.grid_dims,
                                band=pipe.gen_band, bricks=pipe.bricks, ess_max=pipe.ess_max,
                                cells=pipe.cells, sub=pipe.sub, rows=pipe.gen_range)
            gen_ms = timed(run_gen, a.reps)
            # exchange: pack this rank's rows, unpack N shards of its size
            enc_ms = dec_ms = 0.0
            packed = 0
            if world > 1 and getattr(pipe, "packed", None) is not None:
                px = pipe.packed
                enc_ms = timed(lambda: _capi.check(L.vdi_encode_vdi1(px.args, dv.stream_handle())),
                               a.reps)
                packed = int(px.len.item())
                cq = torch.empty_like(pipe.bufs.counts)
                sq = torch.empty_like(pipe.bufs.segs)

                def dec():
                    for _ in range(world):
                        _capi.check(L.vdi_decode_vdi1_lists(
                            dv.ptr(px.buf), pipe.w, pipe.gen_rows, n_sg, dv.ptr(cq), dv.ptr(sq),
                            dv.ptr(px.dec_ws), int(px.dec_ws.numel()), dv.stream_handle()))
                dec_ms = timed(dec, a.reps)
            # this rank's output rows over the full VDI
            img = torch.empty((pipe.out_rows, ow, 4), dtype=torch.float64, device="cuda")
            ra = render_args(full_vdi, n_sg, w, h, gcam, pipe.aabb, ref_grid, pipe.grid_dims,
                             gcam.near, gcam.far, rcam, pipe.opts, img, band=pipe.band)
            zm = alloc_zmask(pipe.grid_dims)

            def run_render():
                launch_zmask(ra, zm)
                _capi.check(L.vdi_render_launch(ra, dv.stream_handle()))
            ren_ms = timed(run_render, a.reps)
            slab_bytes = (pipe.slab_local.numel() * pipe.slab_local.element_size()
                          if pipe.slabs is not None else 0)
            ranks.append({"rank": r, "prep": prep_ms, "gen": gen_ms, "encode": enc_ms,
                          "decode": dec_ms, "render": ren_ms, "packed_bytes": packed,
                          "slab_bytes": slab_bytes, "gen_rows": pipe.local_gen_rays // w,
                          "resident_MB": pipe.vol_dev.numel() * pipe.vol_dev.element_size() / 1e6})
            del pipe
        kern = [x["prep"] + x["gen"] + x["encode"] + x["decode"] + x["render"] for x in ranks]
        gx, gy, gz = ref.grid_dims
        coll = {
            "bricks_allgather": coll_ms(world * max(x["slab_bytes"] for x in ranks), world,
                                        "allgather") if not a.bricked else 0.0,
            "grid_allreduce": coll_ms(4 * gx * gy * gz, world, "allreduce"),
            "lens_allgather": coll_ms(8 * world, world, "allgather"),
            "vdi_allgather": coll_ms(world * max(x["packed_bytes"] for x in ranks), world,
                                     "allgather"),
            "image_allgather": coll_ms(world * shard.rows_per_rank(oh, world) * ow * 32, world,
                                       "allgather"),
        }
        step = max(kern) + sum(coll.values())
        if base_step is None:
            base_step = step
        line = {"config": a.config, "bricked": a.bricked, "balanced": a.balanced,
                "world": world,
                "step_ms": step, "kernels_ms_max": max(kern), "kernels_ms_min": min(kern),
                "imbalance": max(kern) / max(min(kern), 1e-9), "collectives_ms": coll,
                "projected_speedup": base_step / step, "ranks": ranks}
        rows_out.append(line)
        print(json.dumps(line), flush=True)
    print("\n| N | slowest rank kernels ms | fastest | collectives ms (model) | step ms | "
          "projected speed-up |")
    print("|---|---|---|---|---|---|")
    for x in rows_out:
        print(f"| {x['world']} | {x['kernels_ms_max']:.2f} | {x['kernels_ms_min']:.2f} | "
              f"{sum(x['collectives_ms'].values()):.3f} | {x['step_ms']:.2f} | "
              f"{x['projected_speedup']:.2f}x |")


if __name__ == "__main__":
    main()
