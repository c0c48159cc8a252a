"""Parity comparators (TEST INFRASTRUCTURE ONLY): the B200 outputs against the
oracle's on the same inputs, reported as numbers so tests can gate on them
and bench.py can print them. Only tests/ and bench.py's CPU legs import this.

Gates (BASELINE.json north_star): per-ray counts bit-exact on >= 99.9 % of
rays, supersegment depths within 1e-5, composited RGBA within 1e-3; the
render counters (R's RenderStats, raycast.py:39-43, plus lists searched) are
compared per pixel.
"""

from __future__ import annotations

import numpy as np

COUNT_FRAC = 0.999
DEPTH_TOL = 1e-5
RGBA_TOL = 1e-3


def generation(ref: dict, counts, segs, passes=None, samples=None, gammas=None) -> dict:
    """ref: oracle.generate() output restricted to the same rays as counts
    (rows, W) / segs (rows, W, n_sg, 6) AoS. Returns the parity block."""
    counts = np.asarray(counts)
    segs = np.asarray(segs, np.float32)
    same = counts == ref["counts"]
    n_sg = segs.shape[2]
    valid = (np.arange(n_sg)[None, None, :] < ref["counts"][:, :, None]) & same[:, :, None]
    out = {"rays": int(counts.size), "counts_equal_frac": float(same.mean()),
           "count_mismatches": int((~same).sum()),
           "max_depth_diff": 0.0, "max_rgba_diff": 0.0,
           "segs_bit_exact": bool(np.array_equal(segs.view(np.uint32)[same],
                                                 ref["segs"].view(np.uint32)[same]))}
    if valid.any():
        out["max_depth_diff"] = float(np.abs(segs[..., :2] - ref["segs"][..., :2])[valid].max())
        out["max_rgba_diff"] = float(np.abs(segs[..., 2:] - ref["segs"][..., 2:])[valid].max())
    if passes is not None:
        out["passes_equal"] = bool(np.array_equal(np.asarray(passes), ref["passes"]))
    if samples is not None:
        out["samples_equal"] = bool(np.array_equal(np.asarray(samples, np.int64),
                                                   ref["samples"]))
    if gammas is not None:
        out["gammas_bit_exact"] = bool(np.array_equal(
            np.asarray(gammas, np.float64).view(np.uint64), ref["gammas"].view(np.uint64)))
    out["ok"] = bool(out["counts_equal_frac"] >= COUNT_FRAC and out["max_depth_diff"] <= DEPTH_TOL
                     and out["max_rgba_diff"] <= RGBA_TOL)
    return out


def render(ref: dict, image, lists_visited=None, segs_intersected=None,
           lists_searched=None, rows=None) -> dict:
    """ref: oracle.render() output; image (h, w, 4) f64 and per-pixel counters
    of the B200 render; rows: the rows to compare (default all)."""
    sel = slice(None) if rows is None else np.asarray(rows)
    img = np.asarray(image)[sel]
    diff = float(np.abs(img - ref["image"][sel]).max()) if img.size else 0.0
    out = {"pixels": int(img.shape[0] * img.shape[1]) if img.ndim == 3 else 0,
           "max_rgba_diff": diff}
    eq = True
    for name, arr in (("lists_visited", lists_visited), ("segs_intersected", segs_intersected),
                      ("lists_searched", lists_searched)):
        if arr is None:
            continue
        a = np.asarray(arr, np.int64)[sel]
        r = ref[name][sel]
        out[f"{name}_equal"] = bool(np.array_equal(a, r))
        out[f"{name}_total"] = int(r.sum())
        eq &= out[f"{name}_equal"]
    out["counters_equal"] = bool(eq)
    out["ok"] = bool(diff <= RGBA_TOL and eq)
    return out
