"""The multi-rank exchange on one GPU: two ranks (processes) share cuda:0,
collectives over gloo (a plumbing check: no kernel waits on another rank).
Each rank generates its bands, the ranks exchange the VDI -- packed VDI1
shards (shard.PackedExchange, the default) or the padded list-SoA -- and the
gathered VDI, the all-reduced AccelGrid and the gathered image must equal the
single-rank pipeline bit for bit on every rank."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def rank_main(rank, world, port, packed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2206_08660_b200 import shard, synth
        from paper_2206_08660_b200.tuning import TUNING
        TUNING.packed_exchange = bool(packed)
        from paper_2206_08660_b200.generate import GenParams
        from paper_2206_08660_b200.vdi import Vdi
        vol, tf, gcam, rcam, n_sg = synth.config("C2")
        params = GenParams(n_sg=n_sg)
        ref = shard.Pipeline(vol, tf, gcam, rcam, params)
        ref.step()
        rc, rs, rg = ref.host_vdi()
        rimg = ref.image.cpu().numpy()[:rcam.viewport[1]]
        pipe = shard.Pipeline(vol, tf, gcam, rcam, params, world=world, rank=rank)
        assert (pipe.packed is not None) == packed
        pipe.step()
        torch.cuda.synchronize()
        w, h = gcam.viewport
        vdi = Vdi(w, h, n_sg, None, None, gcam, pipe.aabb, _device=pipe.dvdi)
        ok = (np.array_equal(vdi.counts, rc) and
              np.array_equal(vdi.segs.view(np.uint32), rs.view(np.uint32)) and
              np.array_equal(pipe.bufs.grid.cpu().numpy().view(np.uint32), rg))
        img = shard.unshard_image(pipe.g_image.cpu().numpy(), rcam.viewport[1], world)
        ok = ok and np.array_equal(img.view(np.uint64), rimg.view(np.uint64))
        if packed:
            ok = ok and 0 < pipe.packed.bytes_last < pipe.g_segs.numel() * 4
        with open(f"{out}.{rank}", "w") as f:
            f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("packed", [True, False])
def test_two_rank_exchange_matches_single_rank(tmp_path, packed):
    out = str(tmp_path / "res")
    mp.start_processes(rank_main, args=(2, free_port(), packed, out), nprocs=2,
                       start_method="spawn", join=True)
    for r in range(2):
        assert open(f"{out}.{r}").read() == "ok", r
