"""Generate the golden fixtures that pin the CPU oracle (and, transitively, the GPU path) to the
reference implementation.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports the reference package (/root/reference/pkg/src/splatnav) and runs its own hot-path
code on seeded inputs. The blend uses the reference's compiled Cython kernel, built from its
source by oracle/build_ref.sh into oracle/_ref/. Outputs are compressed .npz files next to this
script. Nothing here is imported at test time. The tests read only the .npz files, because
/root/reference does not exist on the GPU box.

Harness-only extractions (the reference computes these but does not return them):
* ids in depth order: np.lexsort is intercepted inside projection.project_cloud, so the ids
  are the reference's own `idx[order]` (projection.py:184);
* tile CSR: renderer._bin_tiles on the reference's projection outputs (renderer.py:80-101);
* per-pixel contributor/visited counts: the oracle's instrumented restatement of the blend loop
  (_kernels_cy.pyx:64-85). This script first asserts that the oracle's accumulators are
  bit-identical to the reference kernel's on the same inputs, so the counts belong to the
  reference's own sequence of decisions.
"""

import hashlib
import importlib.util
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import splatnav  # noqa: E402  (the reference)
from splatnav import projection as ref_projection  # noqa: E402
from splatnav import raster as ref_raster  # noqa: E402
from splatnav import renderer as ref_renderer  # noqa: E402
from splatnav import rig as ref_rig  # noqa: E402
from splatnav.camera import Camera as RefCamera  # noqa: E402
from splatnav.camera import pose_world_to_camera as ref_pose  # noqa: E402
from splatnav.synthetic import make_avatar_bundle, random_cloud  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2604_12626_b200 import synthetic as S  # noqa: E402


def _load_ref_cython():
    ref_dir = os.path.join(REPO, "oracle", "_ref")
    for f in os.listdir(ref_dir) if os.path.isdir(ref_dir) else []:
        if f.startswith("_kernels_cy") and f.endswith(".so"):
            spec = importlib.util.spec_from_file_location("_kernels_cy", os.path.join(ref_dir, f))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    raise SystemExit("build the reference kernel first: oracle/build_ref.sh")


CY = _load_ref_cython()
ref_raster._KERNELS["cython"] = CY  # the reference's own registry (raster/__init__.py:17-19)


def ref_project_with_ids(cloud, cam):
    """projection.project_cloud with np.lexsort intercepted to recover idx[order]."""
    real = ref_projection.np
    captured = {}

    class _Np:
        def __getattr__(self, name):
            if name == "lexsort":
                def lexsort(keys):
                    order = real.lexsort(keys)
                    captured["ids"] = np.asarray(keys[0])[order]
                    return order
                return lexsort
            return getattr(real, name)

    ref_projection.np = _Np()
    try:
        out = ref_projection.project_cloud(cloud, cam)
    finally:
        ref_projection.np = real
    return out, captured.get("ids", np.zeros(0, dtype=np.int64))


def cloud_arrays(cloud, prefix=""):
    return {prefix + "positions": np.asarray(cloud.positions), prefix + "sh_coeffs": np.asarray(cloud.sh_coeffs),
            prefix + "opacities": np.asarray(cloud.opacities), prefix + "log_scales": np.asarray(cloud.log_scales),
            prefix + "rotations": np.asarray(cloud.rotations)}


def cam_arrays(cam, prefix="cam_"):
    return {prefix + "intr": np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near, cam.far]),
            prefix + "size": np.array([cam.width, cam.height]), prefix + "w2c": np.asarray(cam.world_to_camera)}


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def render_case(cloud, cam, background, store_inputs=True, frame_dtype=np.float64, full_pairs=True):
    """Reference render of one cloud + all harness extractions, with the oracle pinned on the way."""
    (m2, con, dep, col, al, rad, st), ids = ref_project_with_ids(cloud, cam)
    tiles_x, tiles_y = math.ceil(cam.width / 16), math.ceil(cam.height / 16)
    if dep.size:
        ts, ps = ref_renderer._bin_tiles(m2, rad, tiles_x, tiles_y)
    else:
        ts, ps = np.zeros(tiles_x * tiles_y + 1, dtype=np.int64), np.zeros(0, dtype=np.int32)
    h, w = cam.height, cam.width
    # reference compiled kernel on the reference's own projection/binning outputs
    cacc, aacc, tr, dacc = np.zeros((h, w, 3)), np.zeros((h, w)), np.ones((h, w)), np.zeros((h, w))
    if dep.size:
        CY.blend_tile_range(0, tiles_x * tiles_y, tiles_x, 16, w, h, ts, ps, m2, con, dep, col, al,
                            cacc, aacc, tr, dacc)
    oc, oa, otr, od, contrib, visited = O.blend(tiles_x, 16, w, h, ts, ps, m2, con, dep, col, al)
    for a, b, name in ((cacc, oc, "color_acc"), (aacc, oa, "alpha_acc"), (tr, otr, "trans"), (dacc, od, "depth_acc")):
        if a.tobytes() != b.tobytes():
            raise SystemExit(f"oracle blend loop is not bit-identical to the reference kernel ({name})")
    frame = ref_renderer.rasterize(cloud, cam, background, kernel="cython")
    brute = ref_renderer.rasterize_reference(cloud, cam, background, kernel="cython")
    assert np.array_equal(frame.color, brute.color) and np.array_equal(frame.depth, brute.depth)
    py = ref_renderer.rasterize(cloud, cam, background, kernel="python")
    assert np.abs(py.color - frame.color).max() < 1e-9
    out = {
        "ids": ids.astype(np.int32), "depths": dep, "means2d": m2, "conics": con, "colors": col, "alphas": al,
        "radii": rad, "tile_starts": ts,
        "contrib": contrib.astype(np.int32), "visited": visited.astype(np.int32),
        "color": frame.color.astype(frame_dtype), "alpha": frame.alpha.astype(frame_dtype),
        "depth": frame.depth.astype(frame_dtype),
        "stats": np.array([st.n_input, st.n_culled_depth, st.n_culled_frame, st.n_degenerate, st.n_drawn]),
        "background": np.asarray(background if background is not None else [np.nan] * 3, dtype=np.float64),
        "pairs_digest": np.array(digest(ps.astype(np.int32))), "n_pairs": np.array(ps.size),
    }
    if full_pairs:
        out["pair_splat"] = ps.astype(np.int32)
    else:  # compact large case: discrete outputs + frames only
        for k in ("means2d", "conics", "colors", "alphas", "radii", "alpha"):
            out.pop(k)
        out["contrib"] = contrib.astype(np.uint16)
        out["visited"] = visited.astype(np.uint16)
    out.update(cam_arrays(cam))
    if store_inputs:
        out.update(cloud_arrays(cloud))
    else:
        out["input_digest"] = np.array(digest(*cloud_arrays(cloud).values()))
    return out


def front_camera(size=64):
    return RefCamera.from_hfov(size, size, 90.0, 0.1, 100.0, ref_pose(np.array([-4.0, 0.0, 1.0]), heading=0.0))


def hand_cloud(positions, colors=None, opacity=4.0, scale=0.3, sh_degree=0, rotations=None):
    """Hand-built cloud whose DC term decodes to `colors` (the reference tests' construction)."""
    positions = np.atleast_2d(np.asarray(positions, dtype=np.float64))
    n = positions.shape[0]
    k = (sh_degree + 1) ** 2
    sh = np.zeros((n, k, 3))
    if colors is not None:
        sh[:, 0, :] = (np.atleast_2d(np.asarray(colors, dtype=np.float64)) - 0.5) / 0.28209479177387814
    rot = np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)) if rotations is None else np.atleast_2d(rotations)
    rot = rot / np.linalg.norm(rot, axis=1, keepdims=True)
    return splatnav.GaussianCloud(positions.astype(np.float32), sh.astype(np.float32),
                                  np.full(n, opacity, dtype=np.float32),
                                  np.full((n, 3), np.log(scale), dtype=np.float32),
                                  rot.astype(np.float32)).validate()


def save(name, cases):
    flat = {}
    for i, case in enumerate(cases):
        for k, v in case.items():
            flat[f"{i}/{k}"] = v
    flat["n_cases"] = np.array(len(cases))
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **flat)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB, {len(cases)} cases)")


def gen_c1():
    """Acceptance C1's 20 seeded scenes (test_acceptance.py:44-65 generator and camera)."""
    cam = front_camera(64)
    bg = np.array([0.9, 0.6, 0.3])
    rng = np.random.default_rng(2024)
    cases = []
    for i in range(20):
        degree = i % 4
        n = int(rng.integers(50, 1001))
        cloud = random_cloud(n, seed=1000 + i, sh_degree=degree, box=2.5, center=(0.0, 0.0, 1.0))
        cases.append(render_case(cloud, cam, bg))
    save("c1_scenes", cases)


def gen_edges():
    cam = front_camera(64)
    bg = np.array([1.0, 0.4, 0.1])
    cases = []
    cases.append(render_case(splatnav.empty_cloud(), cam, bg))                       # empty -> background
    cases.append(render_case(hand_cloud([[-2.0, 0.0, 1.0]], [[0.8, 0.3, 0.6]], 9.0, 0.5), cam, bg))  # single
    c = random_cloud(5, seed=22, box=0.5, center=(0, 0, 1))
    c.log_scales[0] = 500.0                                                          # overflow -> degenerate
    c.log_scales[3] = 400.0
    cases.append(render_case(c, cam, bg))
    t = random_cloud(6, seed=6, sh_degree=0, box=1.0, center=(0, 0, 1))
    t.positions = np.array([[-2.0, 0.1, 1.0], [-2.0, 0.0, 1.0], [-3.0, 0.0, 1.0],
                            [-2.0, -0.1, 1.0], [-2.0, 0.0, 1.3], [-3.0, 0.2, 1.0]], dtype=np.float32)
    cases.append(render_case(t, cam, bg))                                            # exact depth ties
    hug = random_cloud(300, seed=7, sh_degree=2, box=0.3, center=(-3.7, 0.0, 1.0))
    cases.append(render_case(hug, cam, bg))                                          # camera-hugging
    off = random_cloud(400, seed=8, sh_degree=1, box=6.0, center=(0.0, 0.0, 1.0))
    off.log_scales[:] = np.log(0.6)
    cases.append(render_case(off, cam, bg))                                          # big, off-screen
    cases.append(render_case(random_cloud(300, seed=9, sh_degree=3, box=2.0, center=(0, 0, 1)), cam, None))  # layer
    wide = RefCamera.from_hfov(72, 40, 75.0, 0.1, 100.0, ref_pose(np.array([-4.0, 0.5, 1.2]), heading=0.1))
    cases.append(render_case(random_cloud(500, seed=10, sh_degree=3, box=2.0, center=(0, 0, 1)), wide, bg))  # ragged
    save("edges", cases)


def gen_config0():
    scene, cam = S.config0()
    ref_cam = RefCamera(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.near, cam.far, cam.world_to_camera)
    ref_cloud = splatnav.GaussianCloud(scene.positions, scene.sh_coeffs, scene.opacities, scene.log_scales,
                                       scene.rotations)
    case = render_case(ref_cloud, ref_cam, np.array([0.0, 0.0, 0.0]), store_inputs=False)
    save("config0", [case])


def gen_room():
    """Config-1 geometry at 1/10 density (100k gaussians in the 8x8x3 m room), two 640x480 envs."""
    box = S.room_box(1_000_000)
    scene = S.make_scene(100_000, box[0], box[1], seed=5)
    cams = S.room_cameras(2, box, seed=6)
    cases = []
    for cam in cams:
        ref_cam = RefCamera(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height, cam.near, cam.far,
                            cam.world_to_camera)
        cases.append(render_case(scene, ref_cam, np.array([1.0, 1.0, 1.0]), store_inputs=False,
                                 frame_dtype=np.float32, full_pairs=False))
    save("room", cases)


def gen_avatars():
    """sample_pose / lbs_deform / render_observation with avatars (rig.py:78-146, renderer.py:169)."""
    cases = []
    walking = make_avatar_bundle(n_gaussians=120, seed=3, waypoints=((0.0, 0.0), (2.0, 0.0)), speed=0.8, fps=30.0)
    s24 = S.make_avatar(3000, seed=11, n_frames=8, floor_lo=(-1.0, -1.0), floor_hi=(1.0, 1.0))
    for bundle, times in ((walking, [0.0, 2.0 / 30.0, 0.51, 1.234, 1e6]), (s24, [0.0, 0.1, 0.137, 0.2])):
        traj = bundle.trajectory
        for t in times:
            pose = ref_rig.sample_pose(traj, t)
            cloud = ref_rig.lbs_deform(bundle, pose)
            cases.append({
                "canon_positions": np.asarray(bundle.canonical.positions),
                "canon_rotations": np.asarray(bundle.canonical.rotations),
                "weights": np.asarray(bundle.lbs_weights), "inv_bind": np.asarray(bundle.inv_bind),
                "traj_quats": traj.quats, "traj_trans": traj.trans, "fps": np.array(traj.fps), "t": np.array(t),
                "pose_quats": np.concatenate([pose.quats, pose.root_quat[None]]),
                "pose_trans": np.concatenate([pose.trans, pose.root_trans[None]]),
                "out_positions": cloud.positions, "out_rotations": cloud.rotations,
            })
    save("lbs", cases)

    # render_observation: small scene + two deformed walking avatars, and a 24-joint avatar
    cam = RefCamera.from_hfov(96, 64, 90.0, 0.1, 100.0, ref_pose(np.array([-2.5, 0.0, 1.0]), heading=0.0))
    bg = np.array([0.2, 0.5, 0.9])
    scene = random_cloud(600, seed=31, sh_degree=3, box=2.0, center=(1.0, 0.0, 1.0))
    a1 = ref_rig.lbs_deform(walking, ref_rig.sample_pose(walking.trajectory, 0.4))
    a2 = make_avatar_bundle(n_gaussians=200, seed=4, waypoints=((0.5, -0.5), (1.0, 0.6)), speed=0.7, fps=30.0)
    a2c = ref_rig.lbs_deform(a2, ref_rig.sample_pose(a2.trajectory, 0.25))
    s24_pose = ref_rig.sample_pose(s24.trajectory, 0.15)
    a3 = ref_rig.lbs_deform(s24, s24_pose)
    obs = []
    for avatars in ([a1, a2c], [a3], []):
        frame = ref_renderer.render_observation(scene, avatars, cam, bg, kernel="cython")
        case = {"color": frame.color, "alpha": frame.alpha, "depth": frame.depth, "background": bg,
                "n_avatars": np.array(len(avatars))}
        case.update(cloud_arrays(scene, "scene_"))
        for i, a in enumerate(avatars):
            case.update(cloud_arrays(a, f"avatar{i}_"))
        case.update(cam_arrays(cam))
        if avatars:
            layer = ref_renderer.rasterize(splatnav.concat_clouds(avatars), cam, None, kernel="cython")
            case.update({"layer_color": layer.color, "layer_alpha": layer.alpha, "layer_depth": layer.depth})
        obs.append(case)
    save("observation", obs)


if __name__ == "__main__":
    gen_c1()
    gen_edges()
    gen_config0()
    gen_room()
    gen_avatars()
