"""Diagnostic: does a device->host copy on another stream overlap sn_render?"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer

E, H, W = 64, 480, 640
box = S.room_box(1_000_000)
scene = S.make_scene(1_000_000, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(4)]
br = BatchRenderer(scene, bundles, background=(1, 1, 1))
cams = S.room_cameras(E, box, seed=5)
times = np.linspace(0, 1, E)
dev = torch.empty((E, H, W, 5), dtype=torch.float32, device="cuda")
host = torch.empty_like(dev, device="cpu").pin_memory()
rs, cs = torch.cuda.Stream(), torch.cuda.Stream()
def run(copy, render, n=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n):
        if copy:
            with torch.cuda.stream(cs): host.copy_(dev, non_blocking=True)
        if render:
            with torch.cuda.stream(rs): br.render(cams, times)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
run(True, True, 2)
print("copy only %.2f ms" % run(True, False))
print("render only %.2f ms" % run(False, True))
print("copy || render %.2f ms" % run(True, True))
# same with the scene-only renderer (no avatar side stream)
br2 = BatchRenderer(br.scene, None, background=(1, 1, 1))
def run2(copy, n=5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n):
        if copy:
            with torch.cuda.stream(cs): host.copy_(dev, non_blocking=True)
        with torch.cuda.stream(rs): br2.render(cams)
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
print("scene render only %.2f ms" % run2(False))
print("copy || scene render %.2f ms" % run2(True))
