"""Diagnostic: the avatar layer's listed (env, tile) pair-list lengths (last 64-env chunk) on the
config 2 and config 4 (1 or 16 avatars) workloads: the tail of the listed layer blend."""
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
for n, a in ((1_000_000, 4), (3_000_000, 1), (3_000_000, 16)):
    box = S.room_box(n)
    scene = S.make_scene(n, box[0], box[1], seed=0)
    bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(a)]
    br = BatchRenderer(scene, bundles, start_offsets=[0.37 * i for i in range(a)], background=(1, 1, 1))
    cams = S.room_cameras(64, box, seed=1000)
    times = np.random.default_rng(2000).uniform(0, 2, 64)
    for _ in range(2):
        br.render(cams, times, views=False)
    torch.cuda.synchronize()
    cap = 1 << 20
    buf = (ctypes.c_uint32 * cap)()
    cnt = ctypes.c_int64(0)
    assert lib.sn_debug_tile_lens(br.context.handle, 1, buf, ctypes.c_int64(cap), ctypes.byref(cnt)) == 0
    L = np.sort(np.frombuffer(buf, dtype=np.uint32)[: cnt.value].astype(np.int64))[::-1]
    tot = L.sum()
    print(f"n={n} avatars={a}: listed tiles {len(L)}, pairs {tot}, mean {L.mean():.0f}, max {L[0]}, "
          f"top-10 {L[:10].tolist()}, share of pairs in the longest 1% tiles {L[:max(1, len(L) // 100)].sum() / tot:.2f}, "
          f"tiles > 1024 pairs {(L > 1024).sum()}")
