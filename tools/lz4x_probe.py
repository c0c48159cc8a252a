"""Time the exact (serial) LZ4 parse on synthetic inputs: random bytes (no
matches: pure batch cost), zeros (one long match), a repeating 6-byte
pattern (dense short matches), checked against the oracle."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2206_08660_b200 import codec  # noqa: E402
from paper_2206_08660_b200 import device as dv  # noqa: E402
from oracle import oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
rng = np.random.default_rng(0)
cases = {"random": rng.integers(0, 256, n, dtype=np.uint8),
         "zeros": np.zeros(n, np.uint8),
         "words": np.frombuffer(rng.integers(0, 8, n // 4 + 1, dtype=np.uint32).astype(np.float32)
                                .tobytes(), np.uint8)[:n].copy()}
for name, arr in cases.items():
    src = dv.to_device(arr)
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dst, ln = codec.compress_device(src, n, exact=True)
        e1.record()
        torch.cuda.synchronize()
    m = int(ln.item())
    got = dv.to_host(dst[:m]).tobytes()
    t0 = time.perf_counter()
    ref = oracle.lz4_compress(arr.tobytes())
    dt = time.perf_counter() - t0
    print(f"{name:7s} n={n} exact {e0.elapsed_time(e1):9.1f} ms  bytes {m}  equal {got == ref}"
          f"  oracle(1 core) {dt * 1e3:8.1f} ms", flush=True)
