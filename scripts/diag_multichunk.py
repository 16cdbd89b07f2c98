"""Diagnostic: sliced vs unsliced renders with the avatar layer over many envs; for differing pixels,
both values next to the oracle's render_observation (which one deviates)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2604_12626_b200 import synthetic as S, rig
from paper_2604_12626_b200.batch import BatchRenderer
box = S.room_box(1_000_000)
scene = S.make_scene(150_000, box[0], box[1], seed=221)
bundles = [S.make_avatar(2000, seed=222 + i, n_frames=8, floor_lo=(2.0, 2.0), floor_hi=(6.0, 6.0)) for i in range(2)]
n_env = 64
cams = S.room_cameras(n_env, box, seed=223, width=96, height=64)
times = np.linspace(0.0, 0.5, n_env)
outs = []
for ns in (0, 30):
    br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.2], background=(0.4, 0.5, 0.6))
    for _ in range(2):
        o = br.render(cams, times, contrib=True, stats=True, views=False, near_slice=ns)
    outs.append({k: v.cpu().numpy() for k, v in o.items() if hasattr(v, "cpu")})
d = np.any(outs[1]["color"] != outs[0]["color"], axis=-1)
for e in sorted(set(np.nonzero(d)[0].tolist())):
    clouds = [rig.AvatarRuntime(b, start_offset=[0.0, 0.2][a]).deformed_cloud(float(times[e])) for a, b in enumerate(bundles)]
    ref = O.render_observation(scene, clouds, cams[e], np.array([0.4, 0.5, 0.6]))
    for (y, x) in list(zip(*np.nonzero(d[e])))[:6]:
        print(f"env {e} px ({y},{x}): unsliced {outs[0]['color'][e, y, x]} d {outs[0]['depth'][e, y, x]:.6f} | sliced "
              f"{outs[1]['color'][e, y, x]} d {outs[1]['depth'][e, y, x]:.6f} | oracle {ref.color[y, x]} d {ref.depth[y, x]:.6f}"
              f" | contrib {outs[0]['contrib_scene'][e, y, x]} {outs[1]['contrib_scene'][e, y, x]} layer {outs[0]['contrib_layer'][e, y, x]}")
