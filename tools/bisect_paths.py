"""Per-level statistics of the gamma bisection paths (generate.py:219-273) on a
config, reconstructed from each ray's final gamma and pass count: the
bisection from [gamma_init, sqrt(3)] visits midpoints, so the final gamma's
position relative to each midpoint gives the decision (D: n < n_sg - delta,
go lower; U: n > n_sg, go higher; =: the window was hit). Used to choose the
speculation shape of the bisect replays.

    python tools/bisect_paths.py --config C3
"""
import argparse
import os
import sys
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

SQ = 1.7320508075688772


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C3")
    a = p.parse_args()
    import paper_2206_08660_b200 as vb
    from paper_2206_08660_b200 import synth
    vol, tf, gcam, rcam, n_sg = synth.config(a.config)
    params = vb.GenParams(n_sg=n_sg)
    vdi, grid, st = vb.generate_vdi(vol, tf, gcam, params, with_stats=True)
    g0 = params.gamma_init
    lvl = Counter()
    hist = Counter(st.passes.ravel().tolist())
    for g, npass in zip(st.gammas.ravel(), st.passes.ravel()):
        if npass < 2:
            continue
        lo, hi = g0, SQ
        for k in range(npass - 1):
            m = 0.5 * (lo + hi)
            if m == g:
                lvl[(k, "=")] += 1
                break
            if g > m:
                lvl[(k, "U")] += 1
                lo = m
            else:
                lvl[(k, "D")] += 1
                hi = m
    print(a.config, "passes histogram", sorted(hist.items()))
    for k in range(12):
        tot = sum(v for (j, c), v in lvl.items() if j == k)
        if tot:
            print(k, tot, {c: round(v / tot, 3) for (j, c), v in lvl.items() if j == k})


if __name__ == "__main__":
    main()
