"""Profiling driver: the 6M-gaussian room (BASELINE config 3 scale), one 64-env chunk, lean
render (no stats / views), three renders (the profiler takes the third)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer

n = int(os.environ.get("N_SCENE", 6_000_000))
box = S.room_box(n)
scene = S.make_scene(n, box[0], box[1], seed=0)
br = BatchRenderer(scene, None, background=(1, 1, 1))
cams = S.room_cameras(64, box, seed=1000)
for _ in range(3):
    br.render(cams, views=False)
torch.cuda.synchronize()
print("ok")
