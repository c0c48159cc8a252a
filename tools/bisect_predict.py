"""Offline study of the bisect-replay speculation shape (analysis only; uses
the oracle's per-pass trace). For every ray that needs the bisection, the
reference's path of (gamma, n) passes is replayed under three policies and
the number of count-only replays is reported:
  tree   : node + both children (2 levels per replay),
  dchain : node -> down -> down below level 6, tree after,
  pred   : node -> predicted -> predicted, directions from a log-linear fit
           n ~ A + B ln(gamma) through the two smallest-gamma exact counts.

    python tools/bisect_predict.py --config C3 --rows 40
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

SQ = 1.7320508075688772


def traces(cfg, nrows):
    import ctypes
    from oracle import oracle
    from paper_2206_08660_b200 import synth
    from paper_2206_08660_b200.generate import GenParams
    vol, tf, gcam, rcam, n_sg = synth.config(cfg)
    p = GenParams(n_sg=n_sg)
    delta, step, lref = p.resolve(vol)
    w, h = gcam.viewport
    rows = np.unique(np.linspace(0, h - 1, nrows).round().astype(np.int32))
    L = oracle.lib()
    f32 = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    L.vdio_generate_trace.argtypes = L.vdio_generate.argtypes + [
        np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
    nr = len(rows)
    tr = np.full((nr * w, 48), np.nan)
    counts = np.zeros((nr, w), np.int32)
    segs = np.zeros((nr, w, n_sg, 6), np.float32)
    g = np.zeros((nr, w)); ps = np.zeros((nr, w), np.int32); sm = np.zeros((nr, w), np.int64)
    m = lambda a: np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))  # noqa: E731
    L.vdio_generate_trace(np.ascontiguousarray(vol.normalized, np.float32), *vol.dims,
                          np.ascontiguousarray(tf.lut, np.float32), tf.lut.shape[0],
                          m(gcam.proj_view()), m(gcam.inv_proj_view()), m(gcam.position),
                          m(vol.aabb), w, h, n_sg, delta, p.epsilon, p.gamma_init, step, lref,
                          rows.ctypes.data_as(ctypes.c_void_p), -nr, 0, counts, segs, g, ps,
                          sm, tr)
    return tr.reshape(nr * w, 24, 2), ps.ravel(), n_sg, delta


def decisions(path, n_sg, delta):
    out = []
    for gam, n in path[1:]:
        if n > n_sg:
            out.append("U")
        elif n < n_sg - delta:
            out.append("D")
        else:
            out.append("=")
            break
    return out


def predict(hist, lo, hi, n_sg, delta):
    """Directions for the next two levels from a log-linear fit."""
    exact = sorted([(g, n) for g, n in hist if n <= n_sg])
    if len(exact) < 2:
        return None
    (g1, n1), (g2, n2) = exact[0], exact[1]
    if g2 <= g1 or n1 <= n2:
        return None
    b = (n1 - n2) / (math.log(g2) - math.log(g1))
    target = n_sg - 0.5 * delta
    gh = math.exp(math.log(g1) - (target - n1) / b)
    dirs = []
    for _ in range(2):
        mid = 0.5 * (lo + hi)
        if gh < mid:
            dirs.append("D")
            hi = mid
        else:
            dirs.append("U")
            lo = mid
    return dirs


def simulate(paths, n_sg, delta, g0):
    res = {"tree": 0, "dchain": 0, "pred": 0, "hybrid": 0}
    for path in paths:
        d = decisions(path, n_sg, delta)
        for pol in res:
            lvl, hist = 0, [tuple(x) for x in path[:1]]
            lo, hi = g0, SQ
            while lvl < len(d):
                res[pol] += 1
                if pol == "tree" or (pol == "dchain" and lvl >= 6):
                    adv = 1 if d[lvl] == "=" else min(2, len(d) - lvl)
                else:
                    if pol == "dchain" or (pol == "hybrid" and lvl < 6):
                        dirs = ["D", "D"]
                    else:
                        dirs = predict(hist, lo, hi, n_sg, delta)
                    if dirs is None:
                        adv = 1 if d[lvl] == "=" else min(2, len(d) - lvl)
                    else:
                        adv = 1
                        if d[lvl] == dirs[0] and lvl + 1 < len(d):
                            adv = 2
                            if d[lvl + 1] == dirs[1] and lvl + 2 < len(d):
                                adv = 3
                for k in range(lvl, min(lvl + adv, len(d))):
                    gm, n = path[k + 1]
                    hist.append((gm, n))
                    if d[k] == "U":
                        lo = gm
                    elif d[k] == "D":
                        hi = gm
                lvl += adv
    return res


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C2")
    p.add_argument("--rows", type=int, default=32)
    a = p.parse_args()
    tr, passes, n_sg, delta = traces(a.config, a.rows)
    paths = []
    for t, np_ in zip(tr, passes):
        if np_ >= 2:
            k = int(np.sum(~np.isnan(t[:, 0])))
            paths.append([tuple(x) for x in t[:k]])
    print(a.config, "rays with bisection:", len(paths))
    print(simulate(paths, n_sg, delta, 1e-5))


if __name__ == "__main__":
    main()


def nosplit_study(cfg, nrows):
    """How many bisection passes have gamma above the ray's no-split bound
    D* = sqrt(max d^2 along the gamma = inf trajectory): those passes' counts
    are the visible-run count V without running them."""
    import ctypes
    from oracle import oracle
    from paper_2206_08660_b200 import synth
    from paper_2206_08660_b200.generate import GenParams
    tr, passes, n_sg, delta = traces(cfg, nrows)
    vol, tf, gcam, rcam, _ = synth.config(cfg)
    p = GenParams(n_sg=n_sg)
    _, step, lref = p.resolve(vol)
    w, h = gcam.viewport
    rows = np.unique(np.linspace(0, h - 1, nrows).round().astype(np.int32))
    L = oracle.lib()
    i64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
    f64 = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
    f32 = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    L.vdio_nosplit.argtypes = [f32, ctypes.c_int, ctypes.c_int, ctypes.c_int, f32, ctypes.c_int,
                               f64, f64, f64, f64, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                               ctypes.c_double, ctypes.c_void_p, ctypes.c_int, i64, f64]
    V = np.zeros(len(rows) * w, np.int64)
    D2 = np.zeros(len(rows) * w)
    m = lambda a: np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))  # noqa: E731
    L.vdio_nosplit(np.ascontiguousarray(vol.normalized, np.float32), *vol.dims,
                   np.ascontiguousarray(tf.lut, np.float32), tf.lut.shape[0], m(gcam.proj_view()),
                   m(gcam.inv_proj_view()), m(gcam.position), m(vol.aabb), w, h, step, lref,
                   rows.ctypes.data_as(ctypes.c_void_p), len(rows), V, D2)
    tot = saved = 0
    for t, np_, v, d2 in zip(tr, passes, V, D2):
        if np_ < 2:
            continue
        k = int(np.sum(~np.isnan(t[:, 0])))
        for gam, n in t[1:k]:
            tot += 1
            if math.sqrt(d2) < gam:
                saved += 1
                assert n == min(v, n_sg + 1) or n == v, (gam, n, v)
    print(cfg, f"bisection passes {tot}, resolved by the no-split bound {saved} "
               f"({100 * saved / max(tot, 1):.1f} %)")
