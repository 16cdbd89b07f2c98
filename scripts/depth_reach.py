"""Diagnostic (library built with -DSN_BLEND_PROF, SPLATNAV_B200_LIB pointing at it): how far into
each env's depth-sorted list the scene blend's tiles reach before every pixel saturates --
log-spaced histogram over tiles of the consumed fraction, plus the tiles whose list ran out with a
live pixel -- and per env the largest fraction. Sizes the near slice of the depth-sliced scene pass."""
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
labels = ["<=0.1%", "<=0.2%", "<=0.5%", "<=1%", "<=2%", "<=5%", "<=10%", "<=20%", "<=50%", "<100%", "ran out live"]
for n, near in ((1_000_000, 0.1), (3_000_000, 0.1), (6_000_000, 0.1), (1_000_000, 0.01)):
    box = S.room_box(n)
    scene = S.make_scene(n, box[0], box[1], seed=0)
    br = BatchRenderer(scene, None, background=(1, 1, 1))
    tot = np.zeros(11)
    for s in range(3):
        cams = S.room_cameras(64, box, seed=10_000 + s, near=near)
        lib.sn_debug_blend_prof(hist, 1)
        lib.sn_debug_env_frac(frac, 1)
        br.render(cams)
        torch.cuda.synchronize()
        lib.sn_debug_blend_prof(hist, 1)
        lib.sn_debug_env_frac(frac, 1)
        tot += np.array(list(hist)[4:15], dtype=np.float64)
    cum = np.cumsum(tot) / tot.sum()
    print(f"N={n} near={near}: cumulative tile fraction " + ", ".join(f"{l} {c:.4f}" for l, c in zip(labels, cum)))
