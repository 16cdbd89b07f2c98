"""Diagnostic: the bench's end-to-end loop with per-step host timings (render call vs waits)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer, HostPipeline

E, H, W = 64, 480, 640
box = S.room_box(1_000_000)
scene = S.make_scene(1_000_000, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(4)]
br = BatchRenderer(scene, bundles, start_offsets=[0.37 * i for i in range(4)], background=(1, 1, 1))
sets = []
for s in range(13):
    cams = S.room_cameras(E, box, seed=10_000 + s * 7)
    sets.append((cams, np.random.default_rng(20_000 + s).uniform(0, 2, E)))
for i in range(3):
    br.render(*sets[i])
torch.cuda.synchronize()
pipe = HostPipeline(br, E, H, W)
pipe.submit(*sets[0]); pipe.wait(); torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(10):
    a = time.perf_counter()
    slot = pipe.i % len(pipe.host)
    if pipe.done[slot] is not None:
        pipe.done[slot].synchronize()
    b = time.perf_counter()
    pipe.done[slot] = None
    pipe.submit(*sets[3 + i])
    c = time.perf_counter()
    print(f"step {i}: wait slot {1e3*(b-a):6.2f} ms  submit {1e3*(c-b):6.2f} ms", flush=True)
pipe.wait()
print(f"total {1e3*(time.perf_counter()-t0)/10:.2f} ms/step")
t0 = time.perf_counter()
for i in range(10):
    br.render(*sets[3 + i])
torch.cuda.synchronize()
print(f"render only {1e3*(time.perf_counter()-t0)/10:.2f} ms/step")
