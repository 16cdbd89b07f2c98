"""Diagnostic: how the avatar layer's tile pairs spread over tiles (config 2, one step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer
from paper_2604_12626_b200.renderer import tile_csr

box = S.room_box(1_000_000)
scene = S.make_scene(1_000_000, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(4)]
br = BatchRenderer(scene, bundles, start_offsets=[0.37 * i for i in range(4)], background=(1.0, 1.0, 1.0))
E = 64
cams = S.room_cameras(E, box, seed=10_000)
times = np.random.default_rng(20_000).uniform(0, 2, E)
out = br.render(cams, times, contrib=True)
torch.cuda.synchronize()
counts = []
for e in range(E):
    ts, _ = tile_csr(1200, pass_id=1, env=e, context=br.context)
    counts.append(np.diff(ts))
c = np.concatenate(counts)
print("tiles", c.size, "empty", int((c == 0).sum()), "pairs", int(c.sum()))
for q in (50, 75, 90, 95, 99, 99.9):
    print(f"p{q}", np.percentile(c, q))
print("max", c.max(), "tiles >256:", int((c > 256).sum()), ">1024:", int((c > 1024).sum()))
cl = out["contrib_layer"].cpu().numpy() if "contrib_layer" in out else None
if cl is not None:
    print("layer contributions/px mean", cl.mean(), "max", cl.max())
