"""Diagnostic: device->host bandwidth and render/copy overlap for the e2e path."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer, HostPipeline

def t_cuda(fn, n=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n

E, H, W = 64, 480, 640
dev = torch.empty((E, H, W, 5), dtype=torch.float32, device="cuda")
host = torch.empty_like(dev, device="cpu").pin_memory()
ms = t_cuda(lambda: host.copy_(dev, non_blocking=True))
print(f"D2H {dev.numel()*4/1e6:.0f} MB pinned: {ms:.2f} ms = {dev.numel()*4/ms/1e6:.1f} GB/s")
ms = t_cuda(lambda: dev.copy_(host, non_blocking=True))
print(f"H2D pinned: {ms:.2f} ms = {dev.numel()*4/ms/1e6:.1f} GB/s")
box = S.room_box(1_000_000)
scene = S.make_scene(1_000_000, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(4)]
br = BatchRenderer(scene, bundles, background=(1, 1, 1))
cams = S.room_cameras(E, box, seed=5)
times = np.linspace(0, 1, E)
print(f"render only: {t_cuda(lambda: br.render(cams, times)):.2f} ms")
print(f"render_to_host (serial): {t_cuda(lambda: br.render_to_host(cams, times)):.2f} ms")
pipe = HostPipeline(br, E, H, W)
def piped():
    pipe.submit(cams, times)
n = 10
pipe.submit(cams, times); pipe.wait(); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n): pipe.submit(cams, times)
pipe.wait()
print(f"pipelined: {(time.perf_counter()-t0)/n*1e3:.2f} ms per step (wall)")
