"""Diagnostic: do two renders on two streams (two contexts, two host threads) overlap into more
throughput than one? Config 2 workload split into halves."""
import os
import sys
import threading

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
E = int(sys.argv[1]) if len(sys.argv) > 1 else 64
K = 8
sets = [(S.room_cameras(E, box, seed=10_000 + s), np.random.default_rng(20_000 + s).uniform(0, 2, E)) for s in range(K + 3)]
br = BatchRenderer(scene, bundles, start_offsets=[0.37 * i for i in range(4)], background=(1.0, 1.0, 1.0))
ctx2 = N.Context()


def run(ctx, cams, times, out):
    return render_frames(br.scene, cams, br.background, avatars=br.avatars, sim_times=times, context=ctx, out=out)


def alloc(n):
    return {"color": torch.empty((n, 480, 640, 3), device="cuda"), "alpha": torch.empty((n, 480, 640), device="cuda"),
            "depth": torch.empty((n, 480, 640), device="cuda")}


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


out1 = alloc(E)
for i in range(3):
    run(br.context, *sets[i], out1)
ms = timed(lambda: [run(br.context, *sets[3 + i], out1) for i in range(K)])
print(f"one context, {E} envs: {E * K / ms * 1e3:.0f} frames/s")

h = E // 2
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
oa, ob = alloc(h), alloc(E - h)


def worker(ctx, stream, lo, hi, out, idx):
    with torch.cuda.stream(stream):
        for i in idx:
            cams, times = sets[i]
            run(ctx, cams[lo:hi], times[lo:hi], out)
        stream.synchronize()


def two(idx):
    t1 = threading.Thread(target=worker, args=(br.context, s1, 0, h, oa, idx))
    t2 = threading.Thread(target=worker, args=(ctx2, s2, h, E, ob, idx))
    t1.start(); t2.start(); t1.join(); t2.join()


two(range(3))
ms = timed(lambda: two(range(3, 3 + K)))
print(f"two contexts x {h} envs, two threads: {E * K / ms * 1e3:.0f} frames/s")
ms = timed(lambda: [run(br.context, sets[3 + i][0][:h], sets[3 + i][1][:h], oa) for i in range(K)])
print(f"one context, {h} envs: {h * K / ms * 1e3:.0f} frames/s")
