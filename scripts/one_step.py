"""One render step of the bench workload (for ncu captures): scene + 4 avatars, E envs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer

E = int(sys.argv[1]) if len(sys.argv) > 1 else 16
box = S.room_box(1_000_000)
scene = S.make_scene(1_000_000, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(4)]
br = BatchRenderer(scene, bundles, background=(1, 1, 1))
cams = S.room_cameras(E, box, seed=10_000)
times = np.linspace(0, 1.9, E)
for _ in range(2):
    br.render(cams, times)
torch.cuda.synchronize()
print("ok")
