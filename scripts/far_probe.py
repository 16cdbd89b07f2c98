"""Diagnostic for the depth-sliced scene pass: renders a config-3 scene (N gaussians, E envs) with
near_slice = NS a few times, then once inside cudaProfilerStart/Stop so an
`ncu --profile-from-start off` launch list covers exactly one steady-state render."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer

n = int(os.environ.get("N", "3000000"))
e = int(os.environ.get("E", "64"))
ns = int(os.environ.get("NS", "-1"))
box = S.room_box(n)
scene = S.make_scene(n, box[0], box[1], seed=0)
br = BatchRenderer(scene, None, background=(1.0, 1.0, 1.0))
cams = S.room_cameras(e, box, seed=1000)
work = np.zeros(12, dtype=np.int64)
for _ in range(3):
    br.render(cams, views=False, near_slice=ns)
torch.cuda.synchronize()
t = time.perf_counter()
torch.cuda.profiler.start()
br.render(cams, views=False, near_slice=ns)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"N={n} E={e} near_slice={ns}: {1e3 * (time.perf_counter() - t):.1f} ms", flush=True)
if os.environ.get("WORK"):
    import ctypes
    from paper_2604_12626_b200 import _native as N
    from paper_2604_12626_b200.renderer import render_frames
    lib = ctypes.CDLL(N.LIB_PATH)
    for mode in (0, ns):
        work = np.zeros(12, dtype=np.int64)
        render_frames(br.scene, cams, br.background, context=br.context, views=False, near_slice=mode, work=work)
        br.context.sync_stats()
        sc = (ctypes.c_uint64 * 2)()
        lib.sn_debug_slice_counts(br.context.handle, sc)
        print(f"near_slice={mode}: visible {work[0]} gathered {work[2]} scanned {work[3]} contributions {work[4]} "
              f"fixups {work[5]} | unfinished tiles {sc[0]} bucket items {sc[1]}", flush=True)
