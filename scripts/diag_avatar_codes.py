import sys, os, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2604_12626_b200 import _native as N, synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer
n = 3_000_000
box = S.room_box(n)
scene = S.make_scene(200_000, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(16)]
br = BatchRenderer(scene, bundles, start_offsets=[0.37 * i for i in range(16)], background=(1, 1, 1))
lib = ctypes.CDLL(N.LIB_PATH)
tot = np.zeros(5, dtype=np.int64)
for s in range(4):
    cams = S.room_cameras(64, box, seed=1000 + s)
    times = np.random.default_rng(2000 + s).uniform(0, 2, 64)
    br.render(cams, times, views=False)
    torch.cuda.synchronize()
    codes = (ctypes.c_uint8 * (64 * 16))()
    lib.sn_debug_avatar_codes(br.context.handle, codes, ctypes.c_int64(64 * 16))
    tot += np.bincount(np.frombuffer(codes, dtype=np.uint8), minlength=5)[:5]
print("codes (test, depth-culled, -, frame-culled, whole-visible):", tot, tot / tot.sum())
