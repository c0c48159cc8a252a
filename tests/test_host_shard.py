"""Multi-rank host logic of the sharded volume prep (CPU; gloo world 2).

With N > 1 ranks and a replicated volume, each rank computes the brick
maxima of a z-slab (shard.brick_slabs) and the ranks all-gather them: the
slabs must tile the brick grid exactly, with each slab computed from voxel
planes that include the bricks' one-voxel trilinear halo, so the gathered
array equals the full-volume computation (checked here with a numpy
restatement of vdi_volume_brick_max standing in for the kernel, and the
all-gather through torch.distributed / gloo as the pipeline does it).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2206_08660_b200 import shard


def brick_max_ref(a, log2=3):
    nz, ny, nx = a.shape
    b = 1 << log2
    out = np.zeros(((nz + b - 1) // b, (ny + b - 1) // b, (nx + b - 1) // b), a.dtype)
    for bz in range(out.shape[0]):
        for by in range(out.shape[1]):
            for bx in range(out.shape[2]):
                out[bz, by, bx] = a[bz * b:min(bz * b + b, nz - 1) + 1,
                                    by * b:min(by * b + b, ny - 1) + 1,
                                    bx * b:min(bx * b + b, nx - 1) + 1].max()
    return out


def volume(nz, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 256, (nz, 12, 20)).astype(np.uint8)
    a[rng.random(a.shape) < 0.8] = 0
    return a


def slab_of(a, world, rank):
    per, nbz, plan = shard.brick_slabs(a.shape[0], world)
    z0, z1, planes = plan[rank]
    out = np.zeros((per,) + brick_max_ref(a[:2]).shape[1:], a.dtype)
    if planes:
        out[:planes] = brick_max_ref(a[z0:z1])[:planes]
    return out, per, nbz


@pytest.mark.parametrize("nz", [2, 9, 16, 17, 24, 63, 795])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_brick_slabs_tile_the_grid(nz, world):
    per, nbz, plan = shard.brick_slabs(nz, world)
    assert nbz == -(-nz // 8) and per * world >= nbz
    assert sum(p for _, _, p in plan) == nbz
    covered = 0
    for z0, z1, planes in plan:
        if planes == 0:
            continue
        assert z0 == covered * 8
        assert z1 == min((covered + planes) * 8 + 1, nz)  # + the halo plane
        covered += planes


@pytest.mark.parametrize("nz", [9, 17, 40, 65])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_slab_maxima_equal_full(nz, world):
    a = volume(nz, nz)
    full = brick_max_ref(a)
    parts = [slab_of(a, world, r)[0] for r in range(world)]
    gathered = np.concatenate(parts)[:full.shape[0]]
    np.testing.assert_array_equal(gathered, full)


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def rank_main(rank, world, port, nz, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = volume(nz, 7)
        local, per, nbz = slab_of(a, world, rank)
        g = torch.empty((world * per,) + local.shape[1:], dtype=torch.uint8)
        dist.all_gather_into_tensor(g, torch.from_numpy(local))
        if rank == 0:
            np.save(out, g.numpy()[:nbz])
    finally:
        dist.destroy_process_group()


def test_slab_allgather_gloo(tmp_path):
    nz = 795 // 8  # a C3-like slab plan, scaled down
    out = str(tmp_path / "g.npy")
    mp.start_processes(rank_main, args=(2, free_port(), nz, out), nprocs=2,
                       start_method="spawn", join=True)
    np.testing.assert_array_equal(np.load(out), brick_max_ref(volume(nz, 7)))
