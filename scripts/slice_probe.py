"""Diagnostic: the bench's config-2 workload (scene + avatars, fresh cameras per step) rendered with
depth slicing forced on (SN_SLICE_MIN=0 in the environment): per step, the render time, the
workspace retries and the sliced renders that fell back to an unsliced re-run (far_short)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12626_b200 import _native as N
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer

n = int(os.environ.get("N", "1000000"))
a = int(os.environ.get("A", "4"))
e = int(os.environ.get("E", "64"))
near = float(os.environ.get("NEAR", "0.1"))
box = S.room_box(n)
scene = S.make_scene(n, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(a)]
br = BatchRenderer(scene, bundles or None, start_offsets=[0.37 * i for i in range(a)] if a else None,
                   background=(1.0, 1.0, 1.0))
lib = ctypes.CDLL(N.LIB_PATH)
sc = (ctypes.c_uint64 * 3)()
for s in range(int(os.environ.get("STEPS", "12"))):
    cams = S.room_cameras(e, box, seed=10_000 + 7 * s, near=near)
    times = np.random.default_rng(20_000 + s).uniform(0.0, 2.0, size=e)
    torch.cuda.synchronize()
    t = time.perf_counter()
    br.render(cams, times if a else None, views=False)
    torch.cuda.synchronize()
    ms = 1e3 * (time.perf_counter() - t)
    lib.sn_debug_slice_counts(br.context.handle, sc)
    print(f"step {s}: {ms:.1f} ms retries {br.context.render_retries()} fallbacks {sc[2]} "
          f"unfinished {sc[0]} items {sc[1]}", flush=True)
