"""Seeded synthetic workloads for the BASELINE.json configs.

The paper's assets (InteriorGS scenes, AnimatableGaussians avatars, GAMMA motion) are not
available, so these generators stand in for them with the shapes, sizes and distributions that
BASELINE.json names:

* scene gaussians: means uniform in a box, log-scales ~ N(-3.5, 0.5) per axis, unit quaternions
  from normalized N(0,1)^4, opacity logits ~ N(0,1), SH degree 3 (DC ~ N(0,0.5), bands 1-3
  ~ N(0,0.05)); float32 storage like the reference's clouds (synthetic.py:28-34 there);
* cameras: 90 deg HFOV pinholes at 1.25 m, random position in the room and random yaw;
* avatars: 24-joint SMPL-like tree, 50k gaussians sampled on a 1.7 m capsule-union body,
  4 nearest joints with Dirichlet(1) weights (stored float32, the bundle file format's precision),
  per-frame joint rotations with axis-angle ~ N(0, 0.3 rad) and random root translations.

Everything is deterministic given the seed (numpy default_rng).
"""

import math

import numpy as np

from .avatar import AvatarBundle, Skeleton, Trajectory
from .camera import Camera, pose_world_to_camera
from .cloud import GaussianCloud, sh_coeff_count
from .transforms import axis_angle_to_quat, quat_multiply, quat_normalize, rotate

ROOM_1M = (np.array([0.0, 0.0, 0.0]), np.array([8.0, 8.0, 3.0]))  # 8 x 8 m floor, 3 m tall


def make_scene(n, lo, hi, seed=0, sh_degree=3):
    """BASELINE config-0/1 gaussian distribution inside the axis-aligned box [lo, hi]."""
    rng = np.random.default_rng(seed)
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    k = sh_coeff_count(sh_degree)
    positions = rng.uniform(lo, hi, size=(n, 3))
    log_scales = rng.normal(-3.5, 0.5, size=(n, 3))
    rotations = quat_normalize(rng.normal(size=(n, 4)))
    opacities = rng.normal(0.0, 1.0, size=n)
    sh = np.empty((n, k, 3))
    sh[:, 0, :] = rng.normal(0.0, 0.5, size=(n, 3))
    if k > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.05, size=(n, k - 1, 3))
    return GaussianCloud(
        positions=positions.astype(np.float32),
        sh_coeffs=sh.astype(np.float32),
        opacities=opacities.astype(np.float32),
        log_scales=log_scales.astype(np.float32),
        rotations=rotations.astype(np.float32),
    ).validate()


def room_box(n_gaussians):
    """Config-3 scaling: keep the 1M-per-(8x8x3 m) density by growing the floor area with N."""
    s = math.sqrt(n_gaussians / 1_000_000)
    lo, hi = ROOM_1M
    return lo.copy(), np.array([hi[0] * s, hi[1] * s, hi[2]])


def config0():
    """Config 0: 20k gaussians in [-2,2]^3, one 256x256 camera at the origin looking down -z."""
    scene = make_scene(20_000, [-2.0, -2.0, -2.0], [2.0, 2.0, 2.0], seed=0)
    w2c = np.diag([1.0, -1.0, -1.0, 1.0])
    cam = Camera.from_hfov(256, 256, 90.0, 0.01, 100.0, w2c)
    return scene, cam


def room_cameras(n_envs, box, seed=1, width=640, height=480, hfov_deg=90.0, near=0.1, far=100.0, mount=1.25):
    """Config-1 env cameras: uniform x,y inside the box floor, uniform yaw, height `mount`."""
    rng = np.random.default_rng(seed)
    lo, hi = box
    cams = []
    for _ in range(n_envs):
        xy = rng.uniform(lo[:2], hi[:2])
        yaw = rng.uniform(-math.pi, math.pi)
        w2c = pose_world_to_camera(np.array([xy[0], xy[1], mount]), yaw)
        cams.append(Camera.from_hfov(width, height, hfov_deg, near, far, w2c))
    return cams


# 24-joint SMPL-like kinematic tree (parents) and a T-pose rest layout, z-up, facing +x, y left.
SMPL_PARENTS = np.array([-1, 0, 0, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 9, 9, 12, 13, 14, 16, 17, 18, 19, 20, 21])
SMPL_REST = np.array([
    [0.00, 0.00, 0.95], [0.00, 0.09, 0.88], [0.00, -0.09, 0.88], [0.00, 0.00, 1.05],
    [0.00, 0.10, 0.50], [0.00, -0.10, 0.50], [0.00, 0.00, 1.18], [0.00, 0.10, 0.08],
    [0.00, -0.10, 0.08], [0.00, 0.00, 1.30], [0.12, 0.10, 0.02], [0.12, -0.10, 0.02],
    [0.00, 0.00, 1.50], [0.00, 0.07, 1.42], [0.00, -0.07, 1.42], [0.00, 0.00, 1.62],
    [0.00, 0.18, 1.42], [0.00, -0.18, 1.42], [0.00, 0.45, 1.42], [0.00, -0.45, 1.42],
    [0.00, 0.70, 1.42], [0.00, -0.70, 1.42], [0.00, 0.78, 1.42], [0.00, -0.78, 1.42],
])
# capsule radius of the bone ending at each child joint
_BONE_RADIUS = np.array([0.0, 0.08, 0.08, 0.12, 0.07, 0.07, 0.13, 0.05, 0.05, 0.13, 0.04, 0.04,
                         0.06, 0.06, 0.06, 0.10, 0.05, 0.05, 0.045, 0.045, 0.04, 0.04, 0.035, 0.035])


def smpl_skeleton():
    return Skeleton(parents=SMPL_PARENTS.copy(), rest_positions=SMPL_REST.copy()).validate()


def _sample_body(rng, n):
    """Points on a capsule-union body: one capsule per bone, area-weighted choice."""
    bones = [(int(SMPL_PARENTS[j]), j) for j in range(1, 24)]
    p0 = np.array([SMPL_REST[p] for p, _ in bones])
    p1 = np.array([SMPL_REST[c] for _, c in bones])
    r = np.array([_BONE_RADIUS[c] for _, c in bones])
    length = np.linalg.norm(p1 - p0, axis=1)
    area = 2 * np.pi * r * length + 4 * np.pi * r * r
    which = rng.choice(len(bones), size=n, p=area / area.sum())
    t = rng.uniform(0.0, 1.0, size=n)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return p0[which] + t[:, None] * (p1[which] - p0[which]) + r[which, None] * d


def random_pose_trajectory(rng, n_frames, fps, floor_lo, floor_hi, sigma=0.3, parents=None, rest=None):
    """Per-frame local axis-angle ~ N(0, sigma) per joint, forward kinematics to world joint
    transforms, plus a random floor translation and yaw for the root (index J). Default skeleton:
    the 24-joint SMPL-like tree."""
    parents = SMPL_PARENTS if parents is None else np.asarray(parents)
    rest = SMPL_REST if rest is None else np.asarray(rest)
    j = parents.shape[0]
    quats = np.zeros((n_frames, j + 1, 4))
    trans = np.zeros((n_frames, j + 1, 3))
    local = axis_angle_to_quat(rng.normal(0.0, sigma, size=(n_frames, j, 3)))
    for f in range(n_frames):
        quats[f, 0] = local[f, 0]
        trans[f, 0] = rest[0]
        for k in range(1, j):
            p = parents[k]
            quats[f, k] = quat_multiply(quats[f, p], local[f, k])
            trans[f, k] = trans[f, p] + rotate(quats[f, p], rest[k] - rest[p])
    yaw = rng.uniform(-math.pi, math.pi, size=n_frames)
    quats[:, j] = np.stack([np.cos(yaw / 2), np.zeros(n_frames), np.zeros(n_frames), np.sin(yaw / 2)], axis=1)
    trans[:, j, :2] = rng.uniform(floor_lo, floor_hi, size=(n_frames, 2))
    return Trajectory(fps=float(fps), quats=quats, trans=trans).validate()


def make_avatar(n_gaussians=50_000, seed=0, n_frames=64, fps=30.0, floor_lo=(0.0, 0.0), floor_hi=(8.0, 8.0),
                sh_degree=3):
    """Config-2 avatar bundle: capsule-union body, 4-nearest-joint Dirichlet(1) skinning weights."""
    rng = np.random.default_rng(seed)
    k = sh_coeff_count(sh_degree)
    pos = _sample_body(rng, n_gaussians)
    dist = np.linalg.norm(pos[:, None, :] - SMPL_REST[None, :, :], axis=2)
    nearest = np.argsort(dist, axis=1, kind="stable")[:, :4]
    w4 = rng.dirichlet(np.ones(4), size=n_gaussians).astype(np.float32).astype(np.float64)
    weights = np.zeros((n_gaussians, 24))
    np.put_along_axis(weights, nearest, w4, axis=1)
    sh = np.empty((n_gaussians, k, 3))
    sh[:, 0, :] = rng.normal(0.0, 0.5, size=(n_gaussians, 3))
    if k > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.05, size=(n_gaussians, k - 1, 3))
    cloud = GaussianCloud(
        positions=pos.astype(np.float32),
        sh_coeffs=sh.astype(np.float32),
        opacities=rng.normal(2.0, 0.5, size=n_gaussians).astype(np.float32),
        log_scales=rng.normal(-4.0, 0.3, size=(n_gaussians, 3)).astype(np.float32),
        rotations=quat_normalize(rng.normal(size=(n_gaussians, 4))).astype(np.float32),
    ).validate()
    inv_bind = np.tile(np.eye(4), (24, 1, 1))
    inv_bind[:, :3, 3] = -SMPL_REST
    traj = random_pose_trajectory(rng, n_frames, fps, np.asarray(floor_lo), np.asarray(floor_hi))
    return AvatarBundle(canonical=cloud, lbs_weights=weights, inv_bind=inv_bind, skeleton=smpl_skeleton(),
                        trajectory=traj).validate()


def smplx_like_skeleton(n_joints=55):
    """The 24-joint tree extended to n_joints (SMPL-X has 55: body, jaw/eyes, 2 x 15 finger joints):
    extra joints hang as short 3-joint chains off the wrists (20, 21) and the head (15)."""
    parents = list(SMPL_PARENTS)
    rest = [list(r) for r in SMPL_REST]
    anchors = [20, 21, 15]
    k = 0
    while len(parents) < n_joints:
        a = anchors[k % 3]
        base = rest[a]
        for d in range(3):
            if len(parents) >= n_joints:
                break
            parents.append(a if d == 0 else len(parents) - 1)
            off = 0.02 * (d + 1)
            rest.append([base[0] + off, base[1] + 0.01 * ((k // 3) - 2), base[2] - 0.01 * d])
        k += 1
    return Skeleton(parents=np.array(parents), rest_positions=np.array(rest)).validate()


def make_dense_avatar(n_gaussians=2_000, n_joints=24, seed=0, n_frames=16, fps=30.0, temperature=0.02,
                      floor_lo=(0.0, 0.0), floor_hi=(8.0, 8.0), sh_degree=1):
    """An avatar whose skinning rows are dense: softmax(-|p - rest_j|^2 / temperature) over every
    joint (the SMPL / SMPL-X style skins the reference's dense N x J blend accepts, rig.py:112-119)."""
    rng = np.random.default_rng(seed)
    skel = smpl_skeleton() if n_joints == 24 else smplx_like_skeleton(n_joints)
    k = sh_coeff_count(sh_degree)
    pos = _sample_body(rng, n_gaussians)
    d2 = ((pos[:, None, :] - skel.rest_positions[None, :, :]) ** 2).sum(axis=2)
    logits = -(d2 - d2.min(axis=1, keepdims=True)) / temperature
    w = np.exp(logits)
    w = np.maximum(w / w.sum(axis=1, keepdims=True), 1e-6)  # every joint nonzero
    w = (w / w.sum(axis=1, keepdims=True)).astype(np.float32).astype(np.float64)
    sh = np.empty((n_gaussians, k, 3))
    sh[:, 0, :] = rng.normal(0.0, 0.5, size=(n_gaussians, 3))
    if k > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.05, size=(n_gaussians, k - 1, 3))
    cloud = GaussianCloud(
        positions=pos.astype(np.float32), sh_coeffs=sh.astype(np.float32),
        opacities=rng.normal(2.0, 0.5, size=n_gaussians).astype(np.float32),
        log_scales=rng.normal(-4.0, 0.3, size=(n_gaussians, 3)).astype(np.float32),
        rotations=quat_normalize(rng.normal(size=(n_gaussians, 4))).astype(np.float32)).validate()
    inv_bind = np.tile(np.eye(4), (n_joints, 1, 1))
    inv_bind[:, :3, 3] = -skel.rest_positions
    traj = random_pose_trajectory(rng, n_frames, fps, np.asarray(floor_lo), np.asarray(floor_hi),
                                  parents=skel.parents, rest=skel.rest_positions)
    return AvatarBundle(canonical=cloud, lbs_weights=w, inv_bind=inv_bind, skeleton=skel,
                        trajectory=traj).validate()


def baseline_config(index, n_envs=None, n_gaussians=None, n_avatars=None, near=0.1, seed=0):
    """Inputs for BASELINE.json configs 1-4 as a dict (scene, cameras, avatars)."""
    defaults = {1: (64, 1_000_000, 0), 2: (64, 1_000_000, 4), 3: (256, 1_000_000, 0), 4: (1024, 3_000_000, 4)}
    e, n, a = defaults[index]
    e = n_envs if n_envs is not None else e
    n = n_gaussians if n_gaussians is not None else n
    a = n_avatars if n_avatars is not None else a
    box = room_box(n)
    scene = make_scene(n, box[0], box[1], seed=seed)
    cams = room_cameras(e, box, seed=seed + 1, near=near)
    avatars = [make_avatar(50_000, seed=seed + 100 + i, floor_lo=box[0][:2], floor_hi=box[1][:2]) for i in range(a)]
    return {"scene": scene, "cameras": cams, "avatars": avatars, "box": box}
