"""Diagnostic: config-2 step time with the avatar layer on materialized tile lists (default) vs
streamed rectangles (binning=0), and per-stage ms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12626_b200 import _native as N
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer
from paper_2604_12626_b200.renderer import render_frames

box = S.room_box(1_000_000)
scene = S.make_scene(1_000_000, box[0], box[1], seed=0)
bundles = [S.make_avatar(50_000, seed=100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(4)]
br = BatchRenderer(scene, bundles, start_offsets=[0.37 * i for i in range(4)], background=(1.0, 1.0, 1.0))
E, K = 64, 8
sets = [(S.room_cameras(E, box, seed=10_000 + s), np.random.default_rng(20_000 + s).uniform(0, 2, E)) for s in range(K + 3)]
out = {"color": torch.empty((E, 480, 640, 3), device="cuda"), "alpha": torch.empty((E, 480, 640), device="cuda"),
       "depth": torch.empty((E, 480, 640), device="cuda")}
for binning in (-1, 0, -1, 0):
    stage = np.zeros(2 * len(N.STAGES))
    for i in range(3):
        render_frames(br.scene, *sets[i][:1], br.background, avatars=br.avatars, sim_times=sets[i][1],
                      context=br.context, binning=binning, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(3, 3 + K):
        render_frames(br.scene, *sets[i][:1], br.background, avatars=br.avatars, sim_times=sets[i][1],
                      context=br.context, binning=binning, out=out, stage_ms=stage)
    e1.record()
    torch.cuda.synchronize()
    br.context.sync_stats()
    ms = e0.elapsed_time(e1) / K
    st = stage.reshape(2, -1) / K
    print(f"binning={binning}: {E / ms * 1e3:.0f} frames/s, layer stages",
          {n: round(float(st[1, j]), 3) for j, n in enumerate(N.STAGES) if st[1, j] > 0})
