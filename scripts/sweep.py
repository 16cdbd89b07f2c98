"""BASELINE configs 1, 3 and 4 on one GPU (the metric is 'RGB-D frames/sec vs gaussian count &
avatar count'): frames/s and per-stage ms for the scene-complexity sweep (250k..6M gaussians, 256
envs) and the avatar-count sweep (3M scene, 0..16 avatars x 50k, 1,024 envs), plus config 1 and the
near=0.01 sensitivity row of config 2. Inputs are seeded synthetic stand-ins (synthetic.py). Each
point: 2 untimed steps (workspace growth), then 3 timed steps with fresh cameras, CUDA events, renders
pipelined through sn_render_async / sn_render_wait as in bench.py (lean path, no harness views);
stage timers from a separate pass with the avatar layer serialized behind the scene pass.
Prints one JSON line per point."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2604_12626_b200 import _native as N
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.batch import BatchRenderer
from paper_2604_12626_b200.renderer import render_frames


NEAR_SLICE = int(os.environ.get("SN_SWEEP_NEAR_SLICE", "-1"))  # -1 auto, 0 off, 1 on, 2..1000 forced fraction


def point(config, n, a, e, near=0.1, steps=3, warm=2, seed=0):
    box = S.room_box(n)
    scene = S.make_scene(n, box[0], box[1], seed=seed)
    bundles = [S.make_avatar(50_000, seed=seed + 100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(a)]
    br = BatchRenderer(scene, bundles or None, start_offsets=[0.37 * i for i in range(a)] if a else None,
                       background=(1.0, 1.0, 1.0))
    sets = [(S.room_cameras(e, box, seed=1000 + s, near=near), np.random.default_rng(2000 + s).uniform(0, 2, e))
            for s in range(warm + steps)]
    stage = np.zeros(2 * len(N.STAGES))
    work = np.zeros(12, dtype=np.int64)
    for s in range(warm + steps):  # untimed: grows the workspace to fit every timed step's views
        br.render(*sets[s], views=False, near_slice=NEAR_SLICE)
    torch.cuda.synchronize()
    shapes = {"color": (e, 480, 640, 3), "alpha": (e, 480, 640), "depth": (e, 480, 640)}
    outs = [{k: torch.empty(v, device="cuda") for k, v in shapes.items()} for _ in range(2)]

    def run(s, wait, **kw):
        cams, times = sets[s]
        return render_frames(br.scene, cams, br.background, avatars=br.avatars, sim_times=times if a else None,
                             context=br.context, stats=False, out=dict(outs[s % 2]), wait=wait, views=False,
                             near_slice=NEAR_SLICE, **kw)

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pending = []  # pipelined like bench.py: queue step s + 1, then check step s
    for s in range(warm, warm + steps):
        run(s, False)
        pending.append(s)
        if len(pending) > 1 and br.context.render_wait():
            raise RuntimeError("workspace grew inside the timed steps; raise the warm-up")
        if len(pending) > 1:
            pending.pop(0)
    while pending:
        if br.context.render_wait():
            raise RuntimeError("workspace grew inside the timed steps; raise the warm-up")
        pending.pop(0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    for s in range(warm, warm + steps):  # stage timers and work counters: a separate, untimed pass
        run(s, True, stage_ms=stage, work=work, serialize=True)
    br.context.sync_stats()
    st = stage.reshape(2, -1) / steps
    names = list(N.STAGES)
    g = lambda p, *ks: float(sum(st[p, names.index(k)] for k in ks))
    w = work.reshape(2, 6) / steps
    return {"config": config, "n_gaussians": n, "n_avatars": a, "envs": e, "near": near, "near_slice": NEAR_SLICE,
            "frames_per_s": e / (ms / 1e3), "ms_per_step": ms,
            "stage_ms": {"preprocess": g(0, "count", "scan", "emit"), "sort": g(0, "depth_sort", "permute"),
                         "blend": g(0, "blend"), "far": g(0, "far"),
                         "avatar_layer": g(1, "pose", "count", "scan", "emit", "depth_sort", "permute",
                                           "pair_scan", "bin_count", "bin_scatter", "ranges", "blend"),
                         "avatar_layer_preprocess": g(1, "pose", "count", "scan", "emit"),
                         "avatar_layer_blend": g(1, "blend"),
                         "composite": g(1, "composite")},
            "visible_per_env": float(w[0, 0] / e), "contributions_per_pixel": float(w[0, 4] / (e * 640 * 480)),
            "fixup_fraction": float(w[0, 5] / (e * 640 * 480)), "render_retries": br.context.render_retries()}


def main():
    pts = [("config1", 1_000_000, 0, 64, 0.1), ("config2", 1_000_000, 4, 64, 0.1),
           ("config2 near=0.01", 1_000_000, 4, 64, 0.01)]
    pts += [("config3", n, 0, 256, 0.1) for n in (250_000, 1_000_000, 3_000_000, 6_000_000)]
    pts += [("config4", 3_000_000, a, 1024, 0.1) for a in (0, 1, 4, 8, 16)]
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for c, n, a, e, near in pts:
        if only and not c.startswith(only):
            continue
        print(json.dumps(point(c, n, a, e, near)), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
