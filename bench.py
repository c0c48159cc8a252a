"""Benchmark: VDI generation + novel-view VDI rendering on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3]
    python bench.py --impl reference ...      # CPU reference arm (oracle port)

Workload (BASELINE.json configs[2], the 1920x1080 config the metric is quoted
on): Kingsnake-shaped 1024x1024x795 u8 volume, 1920x1080 generation viewport,
n_sg 20, generate at azimuth 0 and render a novel view at 15 deg. One step =
one generate_vdi (generation + AccelGrid) + one render_vdi of that VDI; the
rays of a step are the 1920x1080 generation rays plus the 1920x1080 render
rays. Multi-GPU: interleaved 16-row bands of both viewports per rank, NCCL
all-reduce of the grid + all-gather of the VDI between the two passes and an
all-gather of the image rows at the end. The frame is fixed as N grows, so
scaling is "strong".

One JSON line on rank 0 (see the driver contract in the task statement).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "VDI gen & render Mrays/s (fps @1920×1080) at 1/2/4/8 B200; % HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="C3")
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="target CPU time of the bounded cpu_baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=20,
                   help="frames per e2e measurement (the stream's first upload and last "
                        "readback are not overlapped; more frames amortise them)")
    p.add_argument("--bricked", action="store_true",
                   help="C5 placement: contiguous generation bands, each rank keeping only "
                        "its voxel box resident (shard.band_volume_box)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def host_info(threads):
    """CPU model and threading layer of the CPU legs."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "threads": threads, "os_cpu_count": os.cpu_count(),
            "threading_layer": "OpenMP (libgomp), rows split across threads",
            "arm": "oracle/vdi_oracle.c, the C restatement of vdikit's numba kernels "
                   "(bit-identical outputs); on C2 it runs generation in 1.34 s against "
                   "the reference's own numba 7.25 s on 8 threads, so it is a faster "
                   "(conservative) baseline than vdikit itself"}


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- workload

def kernel_metrics(config):
    """Per-kernel ncu metrics of one step of this workload, from the committed
    capture (profiles/*_<config>_kernel_metrics.json, tools/ncu_metrics_json.py):
    actual DRAM bytes, FP64 pipe utilisation, warp execution efficiency."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles",
                                          f"*_{config.lower()}_kernel_metrics.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        return json.load(f), os.path.relpath(files[-1], ROOT)


def workload(name):
    from paper_2206_08660_b200 import synth
    vol, tf, gcam, rcam, n_sg = synth.config(name)
    return vol, tf, gcam, rcam, n_sg


def sample_rows(height, nrows):
    nrows = max(1, min(height, nrows))
    return np.unique(np.linspace(0, height - 1, nrows).round().astype(np.int64))


def cpu_time_sample(vol, tf, gcam, rcam, n_sg, vdi_counts, vdi_segs, grid, rows, threads):
    """Oracle (C port of the reference kernels) on `rows` of both passes."""
    from oracle import oracle
    from paper_2206_08660_b200.generate import GenParams
    params = GenParams(n_sg=n_sg)
    delta, step, lref = params.resolve(vol)
    w, h = gcam.viewport
    norm = vol.data if vol.voxel_type == "u8" else vol.normalized  # (normalised exactly)
    t0 = time.perf_counter()
    g = oracle.generate(norm, tf.lut, gcam.proj_view(), gcam.inv_proj_view(),
                        np.asarray(gcam.position), vol.aabb, w, h, n_sg, delta, params.epsilon,
                        params.gamma_init, step, lref, rows=rows, threads=threads, compact=True)
    t1 = time.perf_counter()
    r = oracle.render(vdi_segs, vdi_counts, gcam.proj_view(), gcam.inv_proj_view(), vol.aabb,
                      rcam.inv_proj_view(), np.asarray(rcam.position), *rcam.viewport, grid,
                      gcam.near, gcam.far, rows=rows, threads=threads)
    t2 = time.perf_counter()
    cpu_time_sample.last = (g, r)  # the outputs, for the parity block
    return t1 - t0, t2 - t1


def calibrated_rows(vol, tf, gcam, rcam, n_sg, counts, segs, grid, threads, seconds, height):
    probe = sample_rows(height, 8)
    tg, tr = cpu_time_sample(vol, tf, gcam, rcam, n_sg, counts, segs, grid, probe, threads)
    per_row = (tg + tr) / len(probe)
    return sample_rows(height, int(seconds / max(per_row, 1e-6)))


# ---------------------------------------------------------------- reference

def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle
    vol, tf, gcam, rcam, n_sg = workload(args.config)
    w, h = gcam.viewport
    threads = os.cpu_count() or 1
    from paper_2206_08660_b200.generate import GenParams
    params = GenParams(n_sg=n_sg)
    delta, step, lref = params.resolve(vol)
    # untimed setup: the full VDI the sampled render rows traverse
    src = vol.data if vol.voxel_type == "u8" else vol.normalized
    ref = oracle.generate(src, tf.lut, gcam.proj_view(), gcam.inv_proj_view(),
                          np.asarray(gcam.position), vol.aabb, w, h, n_sg, delta,
                          params.epsilon, params.gamma_init, step, lref, threads=threads)
    from paper_2206_08660_b200.vdi import default_grid_dims
    pa, pb = oracle.depth_consts(gcam.near, gcam.far)
    grid = oracle.accumulate_grid(ref["counts"], ref["segs"], default_grid_dims(w, h),
                                  gcam.near, gcam.far, pa, pb)
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    rows = calibrated_rows(vol, tf, gcam, rcam, n_sg, ref["counts"], ref["segs"], grid, threads,
                           budget, h)
    times = []
    for i in range(args.warmup + args.steps):
        tg, tr = cpu_time_sample(vol, tf, gcam, rcam, n_sg, ref["counts"], ref["segs"], grid,
                                 rows, threads)
        if i >= args.warmup:
            times.append(tg + tr)
    rays = 2 * len(rows) * w
    t = float(np.mean(times))
    value = rays / t / 1e6
    sample = f"{len(rows)} of {h} rows (every ~{h / len(rows):.1f}th) of both passes per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mrays/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, gcam, n_sg),
        "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads, "kind": "port",
                         "sample": sample, "host": host_info(threads)},
        "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


DESCRIBE = {
    "C1": "64^3 f32 Gaussian blobs",
    "C2": "256^3 f32 Gaussian blobs",
    "C3": "Kingsnake-shaped 1024x1024x795 u8",
    "C4": "Rayleigh-Taylor-shaped 1024^3 f32",
    "C5": "Richtmyer-Meshkov-shaped 2048x2048x1920 u8",
}


def config_dict(args, gcam, n_sg):
    w, h = gcam.viewport
    par = (f"bricked: contiguous generation bands + resident voxel boxes x{args.gpus}"
           if args.bricked else f"ray-band shard x{args.gpus}")
    return {"workload": f"{args.config}: {DESCRIBE.get(args.config, args.config)}, {w}x{h}, "
                        f"n_sg {n_sg}, generate @0deg + render @15deg",
            "rays_per_step": 2 * w * h, "viewport": [w, h], "n_sg": n_sg,
            "parallelism": par, "l2": "256 MiB L2-flush write between timed steps"}


# --------------------------------------------------------------------- B200

def run_b200(args):
    import torch
    import torch.distributed as tdist

    world, rank, local = dist_env()
    # one process per GPU; VDI_DIST_BACKEND=gloo with more ranks than GPUs is a
    # plumbing check of the multi-rank path on one device (collectives on the
    # host, no kernel waits on another rank), never a measurement
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    backend = os.environ.get("VDI_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            tdist.init_process_group(backend)
    from paper_2206_08660_b200 import device as dv
    from paper_2206_08660_b200 import shard
    from paper_2206_08660_b200.generate import GenParams

    vol, tf, gcam, rcam, n_sg = workload(args.config)
    params = GenParams(n_sg=n_sg)
    w, h = gcam.viewport
    box_volume = None
    if args.config == "C5" and args.bricked:
        from paper_2206_08660_b200 import synth
        box_volume = lambda org, size: synth.rm_like(box=(org, size)).device_data  # noqa: E731
    pipe = shard.Pipeline(vol, tf, gcam, rcam, params, world=world, rank=rank,
                          bricked=args.bricked and world > 1, box_volume=box_volume)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")

    def barrier():
        if world > 1:
            tdist.barrier()

    for _ in range(args.warmup):
        pipe.step()
    torch.cuda.synchronize()
    S = pipe.samples_executed()            # this rank's executed samples (R semantics)
    stats = pipe.exact_render_stats()      # this rank's (L, K, L_s), untimed

    clocks = ClockSampler(dev)
    step_ms, prep_ms, gen_ms, grid_ms, coll_ms, ren_ms = [], [], [], [], [], []
    clocks.start()
    for _ in range(args.steps):
        flush.fill_(1)
        barrier()
        torch.cuda.synchronize()
        ev = pipe.step(timed=True)
        torch.cuda.synchronize()
        barrier()
        step_ms.append(ev["step"])
        prep_ms.append(ev["prep"])
        gen_ms.append(ev["gen"])
        grid_ms.append(ev["grid"])
        coll_ms.append(ev["collective"])
        ren_ms.append(ev["render"])
    clk = clocks.stop()

    total = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if world > 1:
        tdist.all_reduce(total, op=tdist.ReduceOp.MAX)
    t_step = float(total.item()) / args.steps / 1e3          # seconds, max over ranks
    rays = 2 * w * h
    value = rays / t_step / 1e6

    # ---- roofline of the dominant kernel (algorithmic bytes / event time)
    gx, gy, gz = pipe.grid_dims
    n_rays_local = pipe.local_gen_rays
    b_gen = 32 * S + n_rays_local * (4 + 24 * n_sg) + 4 * gx * gy * gz
    L, K, Ls = stats
    b_ren = 4 * L + 8 * Ls + 24 * K + 32 * pipe.local_render_pixels
    peak, peak_kind = peaks()
    g_ms, r_ms = float(np.mean(gen_ms)), float(np.mean(ren_ms))
    gen_gbs = b_gen / (g_ms * 1e-3) / 1e9
    ren_gbs = b_ren / (r_ms * 1e-3) / 1e9
    dominant = "vdi_gen" if g_ms >= r_ms else "vdi_render"
    ach = gen_gbs if dominant == "vdi_gen" else ren_gbs
    # the committed ncu capture is of the full-frame (N=1) step
    km, km_src = kernel_metrics(args.config) if world == 1 else (None, None)
    traffic = None
    ncu = None
    if km is not None:
        ks = km["kernels"]
        traffic = (km["gen_dram_bytes"] if dominant == "vdi_gen"
                   else ks.get("render_kernel", {}).get("dram_bytes"))
        ncu = {"source": km_src, "commit": km.get("commit"),
               "dram_frac": (traffic / ((g_ms if dominant == "vdi_gen" else r_ms) * 1e-3)
                             / (peak * 1e9)) if traffic else None,
               "phases": {k: {"ms_ncu": round(v["ms"], 4),
                              "dram_GB": round(v["dram_bytes"] / 1e9, 3),
                              "dram_GBps": round(v["dram_GBps"], 1),
                              "fp64_pipe_pct": round(v["fp64_pipe_pct"], 1),
                              "warp_exec_eff": round(v["warp_exec_efficiency"], 3),
                              "l2_hit_pct": round(v["l2_hit_pct"], 1)}
                          for k, v in ks.items() if v["ms"] > 0.05},
               "binding": "generation: FP64 dependency latency + issue at 16-20 warps/SM "
                          "(fp64 pipe 20-36 %, dram 5-60 % per phase); render: latency of "
                          "its per-list shading chains (dram ~3 %)"}
    roof = {"kernel": dominant, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak, "peak_kind": peak_kind, "traffic": traffic,
            "traffic_note": "actual DRAM bytes of the generation phases (ncu, one step); "
                            "achieved/frac use the algorithmic bytes of SURVEY 8(d)",
            "ncu": ncu,
            "algorithmic_bytes": b_gen if dominant == "vdi_gen" else b_ren,
            "gen": {"ms": g_ms, "bytes": b_gen, "GBps": gen_gbs, "frac": gen_gbs / peak,
                    "samples": S, "Gsamples_per_s": S / (g_ms * 1e-3) / 1e9},
            "render": {"ms": r_ms, "bytes": b_ren, "GBps": ren_gbs, "frac": ren_gbs / peak,
                       "lists_visited": L, "segs_intersected": K, "lists_searched": Ls}}

    # ---- end to end through the public API with host buffers
    # headline: the VDI comes back in the reference's VDI1 wire format
    # (encode_vdi bytes, packed on the device); "dense" reads back the full
    # (H, W, n_sg, 6) array instead, "serial" is one frame at a time
    if args.bricked and world > 1:
        e2e = {"value": None, "unit": "Mrays/s", "h2d_bytes_per_step": None,
               "d2h_bytes_per_step": None,
               "note": "bricked placement: each rank holds only its voxel box; the "
                       "host-volume e2e path streams whole volumes (not built for boxes)"}
    else:
        e2e = pipe.e2e_stream(args.e2e_steps, packed=True)
        e2e["dense"] = pipe.e2e_stream(args.e2e_steps)
        e2e["serial"] = pipe.e2e(min(args.e2e_steps, 3))

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_dict(args, gcam, n_sg),
            "fps": 1.0 / t_step,
            "phases_ms": {"prep": float(np.mean(prep_ms)), "gen": g_ms, "grid": float(np.mean(grid_ms)),
                          "collective": float(np.mean(coll_ms)), "render": r_ms},
            "gen_mrays_s": w * h / (g_ms * 1e-3) / 1e6,
            "render_mrays_s": w * h / (r_ms * 1e-3) / 1e6,
            "roofline": roof, "e2e": e2e, "clocks": clk,
            "gpu_launches": pipe.launches_per_step * args.steps,
        }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], line["parity"] = pipe_cpu_baseline(vol, tf, gcam, rcam, n_sg,
                                                                 pipe, args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def pipe_cpu_baseline(vol, tf, gcam, rcam, n_sg, pipe, args):
    """The oracle on evenly spaced rows of both passes (timed), and the parity
    of those rows: the oracle's generation against the B200's, and the
    oracle's render of the B200's VDI against the B200's render (image and
    per-pixel counters)."""
    from oracle import parity
    threads = os.cpu_count() or 1
    counts, segs, grid = pipe.host_vdi()
    w, h = gcam.viewport
    rows = calibrated_rows(vol, tf, gcam, rcam, n_sg, counts, segs, grid, threads,
                           args.cpu_seconds, h)
    tg, tr = cpu_time_sample(vol, tf, gcam, rcam, n_sg, counts, segs, grid, rows, threads)
    g_ref, r_ref = cpu_time_sample.last
    rays = 2 * len(rows) * w
    img, lv, si, ls = pipe.render_per_pixel()
    gp = parity.generation(g_ref, counts[rows], segs[rows],
                           pipe.bufs.passes.cpu().numpy()[rows],
                           pipe.bufs.samples.cpu().numpy()[rows],
                           pipe.bufs.gammas.cpu().numpy()[rows])
    rp = parity.render(r_ref, img, lv, si, ls, rows=rows)
    par = {"rows": int(len(rows)), "of": int(h),
           "counts_equal_frac": gp["counts_equal_frac"], "segs_bit_exact": gp["segs_bit_exact"],
           "max_depth_diff": gp["max_depth_diff"], "max_seg_rgba_diff": gp["max_rgba_diff"],
           "passes_samples_gammas_equal": bool(gp["passes_equal"] and gp["samples_equal"]
                                               and gp["gammas_bit_exact"]),
           "max_rgba_diff": rp["max_rgba_diff"], "counters_equal": rp["counters_equal"],
           "ok": bool(gp["ok"] and rp["ok"]),
           "note": "oracle generation vs B200 generation on these rows; oracle render of "
                   "the B200 VDI vs the B200 render on these rows (full-frame parity: "
                   "tests/test_gpu_full_c3.py)"}
    return {"value": rays / (tg + tr) / 1e6, "unit": "Mrays/s", "cores": threads,
            "kind": "port",
            "sample": f"{len(rows)} of {h} evenly spaced rows of both passes "
                      f"(gen {tg:.2f} s + render {tr:.2f} s)",
            "host": host_info(threads)}, par


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
