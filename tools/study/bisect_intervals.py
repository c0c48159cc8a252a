"""Offline study driver (tools/study/bisect_intervals.c): fraction of the
bisection passes after pass 1 whose gamma lies in the identical-trajectory
interval of an earlier pass of the same ray (answerable without re-walking
the samples). usage: python tools/study/bisect_intervals.py [C3] [nrows]"""
import ctypes
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_2206_08660_b200 import synth  # noqa: E402
from paper_2206_08660_b200.generate import GenParams  # noqa: E402

so = os.path.join(HERE, "bisect_intervals.so")
subprocess.run(["/usr/bin/gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                "-o", so, os.path.join(HERE, "bisect_intervals.c"), "-lm"], check=True)
L = ctypes.CDLL(so)
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 24
vol, tf, gcam, rcam, n_sg = synth.config(cfg)
params = GenParams(n_sg=n_sg)
delta, step, lref = params.resolve(vol)
w, h = gcam.viewport
rows = np.linspace(0, h - 1, nrows).round().astype(np.int32)
data = np.ascontiguousarray(vol.data if vol.voxel_type == "u8" else vol.normalized)
assert data.dtype == np.uint8, "u8 volumes only in this study"
m = lambda a: np.ascontiguousarray(np.asarray(a, np.float64).reshape(-1))  # noqa: E731
out = np.zeros(3, np.int64)
P = ctypes.c_void_p
L.study_rows(data.ctypes.data_as(P), *(int(v) for v in vol.dims),
             np.ascontiguousarray(tf.lut, np.float32).ctypes.data_as(P), int(tf.lut.shape[0]),
             m(gcam.proj_view()).ctypes.data_as(P), m(gcam.inv_proj_view()).ctypes.data_as(P),
             m(gcam.position).ctypes.data_as(P), m(vol.aabb).ctypes.data_as(P),
             w, h, n_sg, delta, ctypes.c_double(params.epsilon),
             ctypes.c_double(params.gamma_init), ctypes.c_double(step), ctypes.c_double(lref),
             rows.ctypes.data_as(P), len(rows), out.ctypes.data_as(P))
print(f"{cfg} rows {len(rows)}: queued rays {out[2]}, bisection passes after pass 1 {out[0]}, "
      f"answerable from an earlier pass {out[1]} ({100 * out[1] / max(out[0], 1):.1f} %)")
