"""Diagnostic: per-warp blend work counters (library built with -DSN_BLEND_PROF), one bench step."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_12626_b200 import synthetic as S, _native as N
from paper_2604_12626_b200.batch import BatchRenderer

lib = ctypes.CDLL(N.LIB_PATH)
out = (ctypes.c_ulonglong * 16)()
box = S.room_box(1_000_000)
scene = S.make_scene(1_000_000, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(4)]
names = ["warp_iters", "lane_boundary_f64", "lane_t_ambiguous"]
for label, av in (("scene only", []), ("scene+avatars", bundles)):
    br = BatchRenderer(scene, av, background=(1, 1, 1))
    cams = S.room_cameras(64, box, seed=10_000)
    times = np.linspace(0, 1.9, 64)
    br.render(cams, times); torch.cuda.synchronize()
    lib.sn_debug_blend_prof(out, 1)
    br.render(cams, times); torch.cuda.synchronize()
    lib.sn_debug_blend_prof(out, 1)
    v = list(out)
    print(label, {n: v[i] for i, n in enumerate(names)})
