"""Multi-rank host path on CPU (gloo, world size 2).

Each rank computes its bands of the generation and of the render viewport
(here with the CPU oracle standing in for the kernels, which cannot run
without a GPU), then the ranks exchange through the very functions the NCCL
pipeline uses (shard.exchange_vdi / shard.gather_rows). The gathered VDI,
the all-reduced AccelGrid and the gathered image must equal a single-process
run bit for bit.

Layouts: "interleaved" (16-row bands, rank b % world), "bricked"
(contiguous generation bands, each rank sampling a volume in which every
voxel outside its planned resident box, shard.band_volume_box, is poisoned:
any ray that reached outside the box would change the result) and
"balanced" (bricked, with contiguous bands of unequal height from
shard.balance_bands, gathered through shard.row_storage_map).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2206_08660_b200 import shard, synth
from paper_2206_08660_b200.generate import GenParams, list_stride
from paper_2206_08660_b200.vdi import default_grid_dims


def to_list_soa(aos):
    """(..., n_sg, 6) reference layout -> (lists, stride) list-SoA rows
    (include/vdi_b200.h: [rgba float4 x n_sg | front | back | pad])."""
    n_sg = aos.shape[-2]
    flat = aos.reshape(-1, n_sg, 6)
    out = np.zeros((flat.shape[0], list_stride(n_sg)), np.float32)
    out[:, : 4 * n_sg] = flat[:, :, 2:6].reshape(flat.shape[0], -1)
    out[:, 4 * n_sg: 5 * n_sg] = flat[:, :, 0]
    out[:, 5 * n_sg: 6 * n_sg] = flat[:, :, 1]
    return out


def from_list_soa(soa, n_sg):
    aos = np.zeros((soa.shape[0], n_sg, 6), np.float32)
    aos[:, :, 2:6] = soa[:, : 4 * n_sg].reshape(-1, n_sg, 4)
    aos[:, :, 0] = soa[:, 4 * n_sg: 5 * n_sg]
    aos[:, :, 1] = soa[:, 5 * n_sg: 6 * n_sg]
    return aos


def scene():
    vol, tf, gcam, rcam, n_sg = synth.config("C1")
    params = GenParams(n_sg=n_sg)
    delta, step, lref = params.resolve(vol)
    return vol, tf, gcam, rcam, n_sg, (delta, step, lref), params


def gen(vol, tf, cam, n_sg, res, params, rows=None):
    delta, step, lref = res
    w, h = cam.viewport
    return oracle.generate(vol.normalized, tf.lut, cam.proj_view(), cam.inv_proj_view(),
                           np.asarray(cam.position), vol.aabb, w, h, n_sg, delta,
                           params.epsilon, params.gamma_init, step, lref, rows=rows)


def render(counts, segs, vol, gcam, rcam, grid, rows=None):
    return oracle.render(segs, counts, gcam.proj_view(), gcam.inv_proj_view(), vol.aabb,
                         rcam.inv_proj_view(), np.asarray(rcam.position), *rcam.viewport, grid,
                         gcam.near, gcam.far, rows=rows)


def poisoned(vol, box):
    """vol with every voxel outside box = (origin, size) set to 1.0."""
    from paper_2206_08660_b200.volume import make_volume
    (ox, oy, oz), (sx, sy, sz) = box
    data = np.ones_like(vol.normalized)
    data[oz:oz + sz, oy:oy + sy, ox:ox + sx] = vol.normalized[oz:oz + sz, oy:oy + sy,
                                                             ox:ox + sx]
    return make_volume(data, "f32")


def rank_main(rank, world, port, out, layout="interleaved"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        vol, tf, gcam, rcam, n_sg, res, params = scene()
        w, h = gcam.viewport
        dims = default_grid_dims(w, h)
        pa, pb = oracle.depth_consts(gcam.near, gcam.far)
        band = -(-h // world) if layout == "bricked" else shard.BAND_ROWS
        mine = shard.band_rows(h, world, rank, band)
        per = shard.rows_per_rank(h, world, band)
        bounds = None
        if layout == "balanced":
            # contiguous bands of unequal height (shard.balance_bands of a
            # per-row cost: here a made-up one that loads the middle rows)
            cost = 1.0 + np.exp(-((np.arange(h) - 0.45 * h) / (0.12 * h)) ** 2) * 50
            bounds = shard.balance_bands(cost, world)
            mine = np.arange(bounds[rank], bounds[rank + 1])
            per = max(bounds[q + 1] - bounds[q] for q in range(world))
            assert len(set(bounds[q + 1] - bounds[q] for q in range(world))) > 1
        gvol = vol
        if layout in ("bricked", "balanced"):
            box = shard.band_volume_box(vol, gcam, int(mine[0]), int(mine[-1]) + 1)
            assert box[1][1] < vol.dims[1]  # a real slab, not the whole volume
            gvol = poisoned(vol, box)
        local = gen(gvol, tf, gcam, n_sg, res, params, rows=mine)
        # local shard, padded to rows_per_rank rows (what the gen kernel writes)
        counts = np.zeros((per, w), np.int32)
        counts[: len(mine)] = local["counts"][mine]
        segs = np.zeros((per * w, list_stride(n_sg)), np.float32)
        segs[: len(mine) * w] = to_list_soa(local["segs"][mine])
        part = oracle.accumulate_grid(local["counts"], local["segs"], dims, gcam.near,
                                      gcam.far, pa, pb)  # only this rank's lists
        t_counts, t_segs = torch.from_numpy(counts), torch.from_numpy(segs)
        t_grid = torch.from_numpy(part.view(np.int32).copy())
        g_counts = torch.empty((world * per, w), dtype=torch.int32)
        g_segs = torch.empty((world * per * w, segs.shape[1]), dtype=torch.float32)
        shard.exchange_vdi(dist, t_counts, t_segs, t_grid, g_counts, g_segs)
        # gathered storage -> natural rows (the render kernel reads the
        # storage rows through the same maps)
        st = (shard.storage_rows(h, world, band) if bounds is None
              else shard.row_storage_map(bounds, per))
        full_counts = g_counts.numpy()[st]
        full_segs = from_list_soa(g_segs.numpy().reshape(world * per, w, -1)[st].reshape(h * w, -1),
                                  n_sg).reshape(h, w, n_sg, 6)
        grid = t_grid.numpy().view(np.uint32)
        # render this rank's output bands over the gathered VDI
        ow, oh = rcam.viewport
        orows = shard.band_rows(oh, world, rank)
        oper = shard.rows_per_rank(oh, world)
        r = render(full_counts, full_segs, vol, gcam, rcam, grid, rows=orows)
        img = np.zeros((oper, ow, 4), np.float64)
        img[: len(orows)] = r["image"][orows]
        g_img = shard.gather_rows(dist, torch.from_numpy(img), world, oper)
        image = g_img.numpy()[shard.storage_rows(oh, world)]
        if rank == 0:
            np.savez(out, counts=full_counts, segs=full_segs, grid=grid, image=image)
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,layout", [(2, "interleaved"), (2, "bricked"),
                                          (2, "balanced"), (3, "balanced")])
def test_sharded_generate_render_equals_single_process(tmp_path, world, layout):
    out = str(tmp_path / "rank0.npz")
    mp.start_processes(rank_main, args=(world, free_port(), out, layout), nprocs=world,
                       start_method="spawn", join=True)
    got = np.load(out)
    vol, tf, gcam, rcam, n_sg, res, params = scene()
    ref = gen(vol, tf, gcam, n_sg, res, params)
    pa, pb = oracle.depth_consts(gcam.near, gcam.far)
    grid = oracle.accumulate_grid(ref["counts"], ref["segs"], default_grid_dims(*gcam.viewport),
                                  gcam.near, gcam.far, pa, pb)
    assert np.array_equal(got["counts"], ref["counts"])
    assert np.array_equal(got["segs"].view(np.uint32), ref["segs"].view(np.uint32))
    assert np.array_equal(got["grid"], grid)
    img = render(ref["counts"], ref["segs"], vol, gcam, rcam, grid)["image"]
    assert np.array_equal(got["image"].view(np.uint64), img.view(np.uint64))
