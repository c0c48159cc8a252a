"""Time the device wire path on a config's VDI: VDI1 packing
(vdi_encode_vdi1) and LZ4 (vdi_lz4_compress, the chunk-parallel parse, and
vdi_lz4_compress_exact, the reference's serial parse), device resident, CUDA events,
median of --reps. Prints one JSON line with GB/s of raw VDI1 bytes, the
compression ratio, and (with --cpu) the reference's serial compressor (the
pinned C restatement of lz4.py:51-114, one core as in the reference) and the
numpy VDI1 packing on the host for the CPU baseline.

    python tools/bench_codec.py --config C3 [--reps 5] [--cpu]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2206_08660_b200 as vb  # noqa: E402
from paper_2206_08660_b200 import codec, synth  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C3")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--cpu", action="store_true")
    a = p.parse_args()
    vol, tf, gcam, rcam, n_sg = synth.config(a.config)
    vdi, grid = vb.generate_vdi(vol, tf, gcam, vb.GenParams(n_sg=n_sg))
    raw, raw_len = codec.encode_vdi_device(vdi, grid)
    torch.cuda.synchronize()
    n = int(raw_len.item())
    enc_ms = timed(lambda: codec.encode_vdi_device(vdi, grid), a.reps)
    comp, clen = codec.compress_device(raw, int(raw.numel()), raw_len, exact=False)
    torch.cuda.synchronize()
    m = int(clen.item())
    lz_ms = timed(lambda: codec.compress_device(raw, int(raw.numel()), raw_len, exact=False),
                  a.reps)
    xcomp, xlen = codec.compress_device(raw, int(raw.numel()), raw_len, exact=True)
    torch.cuda.synchronize()
    mx = int(xlen.item())
    lzx_ms = timed(lambda: codec.compress_device(raw, int(raw.numel()), raw_len, exact=True),
                   max(1, a.reps // 2))
    line = {"tool": "bench_codec", "config": a.config, "raw_bytes": n, "lz4_bytes": m,
            "ratio": n / max(m, 1), "encode_ms": enc_ms, "encode_GBps": n / enc_ms / 1e6,
            "lz4_ms": lz_ms, "lz4_GBps": n / lz_ms / 1e6,
            "lz4_exact": {"ms": lzx_ms, "bytes": mx, "ratio": n / max(mx, 1),
                          "GBps": n / lzx_ms / 1e6},
            "counts_segs_read_bytes": 4 * vdi.width * vdi.height + 24 * (n - 160) // 26}
    if a.cpu:
        from oracle import oracle
        host = dv.to_host(raw[:n]).tobytes()
        t0 = time.perf_counter()
        ref = oracle.lz4_compress(host)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"lz4_ms": dt * 1e3, "lz4_bytes": len(ref),
                                "ratio": n / max(len(ref), 1), "cores": 1, "kind": "port",
                                "sample": "the whole VDI1 stream, reference serial parse"}
        assert oracle.lz4_decompress(dv.to_host(comp[:m]).tobytes(), n) == host
        line["lz4_exact"]["equals_reference"] = dv.to_host(xcomp[:mx]).tobytes() == ref
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
