"""Diagnostic: how the scene pass's float64 fixup pixels spread over (env, tile) on the bench
workload (one 64-env chunk): pixels per tile with any, and their list positions."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12626_b200 import _native as N
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer

n = 1_000_000
box = S.room_box(n)
scene = S.make_scene(n, box[0], box[1], seed=0)
br = BatchRenderer(scene, None, background=(1, 1, 1))
cams = S.room_cameras(64, box, seed=10_000)
for _ in range(2):
    br.render(cams, views=False)
torch.cuda.synchronize()
lib = ctypes.CDLL(N.LIB_PATH)
cap = 1 << 22
buf = (ctypes.c_uint32 * cap)()
cnt = ctypes.c_int64(0)
assert lib.sn_debug_fix_list(br.context.handle, 0, buf, ctypes.c_int64(cap), ctypes.byref(cnt)) == 0
codes = np.frombuffer(buf, dtype=np.uint32)[: min(cnt.value, cap)]
W, H = 640, 480
el, p = codes // (W * H), codes % (W * H)
tile = (p // W // 16) * (W // 16) + (p % W) // 16
key = el.astype(np.int64) * 10_000 + tile
u, c = np.unique(key, return_counts=True)
print(f"fixup pixels {cnt.value}, (env, tile)s with any {len(u)}, pixels per such tile: mean {c.mean():.2f}, "
      f"median {np.median(c):.0f}, max {c.max()}")
print("histogram (1, 2, 3-4, 5-8, 9-16, 17-64, >64):",
      [int(((c >= lo) & (c <= hi)).sum()) for lo, hi in ((1, 1), (2, 2), (3, 4), (5, 8), (9, 16), (17, 64), (65, 1 << 30))])
print("share of pixels in tiles with >= 8:", float(c[c >= 8].sum()) / max(1, c.sum()))
