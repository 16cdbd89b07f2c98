"""Diagnostic (library built with -DSN_BLEND_PROF): how far into each env's depth-sorted list the
scene blend's tiles reach before every pixel saturates. Histogram over tiles of the consumed
fraction, and per env the largest fraction."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12626_b200 import _native as N
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer

lib = ctypes.CDLL(N.LIB_PATH)
hist = (ctypes.c_ulonglong * 16)()
frac = (ctypes.c_uint * 64)()
for n, near in ((1_000_000, 0.1), (6_000_000, 0.1), (1_000_000, 0.01)):
    box = S.room_box(n)
    scene = S.make_scene(n, box[0], box[1], seed=0)
    br = BatchRenderer(scene, None, background=(1, 1, 1))
    for s in range(2):
        cams = S.room_cameras(64, box, seed=10_000 + s, near=near)
        lib.sn_debug_blend_prof(hist, 1)
        lib.sn_debug_env_frac(frac, 1)
        br.render(cams)
        torch.cuda.synchronize()
        lib.sn_debug_blend_prof(hist, 1)
        lib.sn_debug_env_frac(frac, 1)
        h = np.array(list(hist)[4:16], dtype=np.float64)
        f = np.array(list(frac)) / 1000.0
        print(f"N={n} near={near} step {s}: tiles by consumed fraction (12 bins) {np.round(h / h.sum(), 4).tolist()}")
        print(f"   per-env max fraction: min {f.min():.3f} median {np.median(f):.3f} max {f.max():.3f}")
