"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper around the CPU oracle (splat_oracle.c).

This is the parity checker for the B200 path, not part of the product. Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may import it. The product package
(``paper_2604_12626_b200``) never does.

Functions mirror the reference's hot-path entry points (``/root/reference/pkg/src/splatnav``):
``project_cloud`` (projection.py:100), ``bin_tiles`` (renderer.py:80), ``rasterize`` /
``rasterize_reference`` (renderer.py:135,145), ``composite`` (renderer.py:151),
``render_observation`` (renderer.py:169), ``sample_pose`` (rig.py:78), ``lbs_deform``
(rig.py:107). They also return harness-only extras the reference computes but does not
expose: original ids in depth order, the tile CSR, and per-pixel contributor/visited counts.

Inputs are duck-typed. A cloud has .positions/.sh_coeffs/.opacities/.log_scales/.rotations.
A camera has .fx/.fy/.cx/.cy/.width/.height/.near/.far/.world_to_camera. Reference objects and
the product's own containers both work.
"""

import ctypes
import math
import os
import subprocess
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

TILE_SIZE = 16


class OrCamera(ctypes.Structure):
    _fields_ = [
        ("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
        ("near_", ctypes.c_double), ("far_", ctypes.c_double),
        ("rot", ctypes.c_double * 9), ("trans", ctypes.c_double * 3), ("center", ctypes.c_double * 3),
        ("background", ctypes.c_double * 3),
        ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("has_background", ctypes.c_int32),
        ("pad", ctypes.c_int32),
    ]


class OrStats(ctypes.Structure):
    _fields_ = [("n_input", ctypes.c_int64), ("n_culled_depth", ctypes.c_int64),
                ("n_culled_frame", ctypes.c_int64), ("n_degenerate", ctypes.c_int64),
                ("n_drawn", ctypes.c_int64)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class OrCloud(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("K", ctypes.c_int32),
                ("pos", ctypes.c_void_p), ("ls", ctypes.c_void_p), ("rot", ctypes.c_void_p),
                ("opac", ctypes.c_void_p), ("sh", ctypes.c_void_p)]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.or_project.restype = ctypes.c_int64
        L.or_project.argtypes = [ctypes.c_int64, P, P, P, P, P, ctypes.c_int, ctypes.POINTER(OrCamera),
                                 P, P, P, P, P, P, P, ctypes.POINTER(OrStats)]
        L.or_count_pairs.restype = ctypes.c_int64
        L.or_count_pairs.argtypes = [ctypes.c_int64, P, P, ctypes.c_int, ctypes.c_int]
        L.or_bin_tiles.restype = None
        L.or_bin_tiles.argtypes = [ctypes.c_int64, P, P, ctypes.c_int, ctypes.c_int, P, P]
        L.or_blend.restype = None
        L.or_blend.argtypes = [ctypes.c_int] * 6 + [P] * 13
        L.or_rasterize.restype = ctypes.c_int64
        L.or_rasterize.argtypes = [ctypes.POINTER(OrCloud), ctypes.POINTER(OrCamera), ctypes.c_int, ctypes.c_int,
                                   P, P, P, P, P, ctypes.POINTER(OrStats)]
        L.or_composite.restype = None
        L.or_composite.argtypes = [ctypes.c_int64] + [P] * 9
        L.or_sample_pose.restype = ctypes.c_int
        L.or_sample_pose.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, P, P, ctypes.c_double, P, P]
        L.or_lbs_deform.restype = None
        L.or_lbs_deform.argtypes = [ctypes.c_int64, ctypes.c_int, P, P, P, P, P, P, P, P]
        L.or_render_batch.restype = None
        L.or_render_batch.argtypes = [ctypes.POINTER(OrCloud), ctypes.POINTER(OrCloud), ctypes.POINTER(OrCamera),
                                      ctypes.c_int, ctypes.c_int, P, P, P]
        _lib = L
    return _lib


def _f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def camera_center(w2c):
    """camera.py:43-48 verbatim arithmetic (numpy matvec), so the oracle sees the same centre."""
    r = w2c[:3, :3]
    t = w2c[:3, 3]
    return -r.T @ t


def make_camera(cam, background=None):
    w2c = np.asarray(cam.world_to_camera, dtype=np.float64)
    c = OrCamera()
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.near_, c.far_ = float(cam.near), float(cam.far)
    for i in range(9):
        c.rot[i] = float(w2c[i // 3, i % 3])
    for i in range(3):
        c.trans[i] = float(w2c[i, 3])
    center = camera_center(w2c)
    for i in range(3):
        c.center[i] = float(center[i])
    c.width, c.height = int(cam.width), int(cam.height)
    if background is None:
        c.has_background = 0
    else:
        bg = np.asarray(background, dtype=np.float64)
        for i in range(3):
            c.background[i] = float(bg[i])
        c.has_background = 1
    return c


class _CloudArrays:
    """Keeps float64 copies alive while the C side holds pointers."""

    def __init__(self, cloud):
        n = int(np.asarray(cloud.positions).shape[0])
        self.n = n
        sh = np.asarray(cloud.sh_coeffs)
        self.K = int(sh.shape[1]) if sh.ndim == 3 else 1
        self.pos = _f64(cloud.positions, (n, 3))
        self.ls = _f64(cloud.log_scales, (n, 3))
        self.rot = _f64(cloud.rotations, (n, 4))
        self.opac = _f64(cloud.opacities, (n,))
        self.sh = _f64(sh, (n, self.K, 3))
        self.c = OrCloud(n, self.K, _ptr(self.pos), _ptr(self.ls), _ptr(self.rot), _ptr(self.opac), _ptr(self.sh))


def project_cloud(cloud, camera):
    """projection.py:100-194. Returns the reference's 6 arrays plus `ids` and `stats`."""
    ca = _CloudArrays(cloud)
    n = max(ca.n, 1)
    out = SimpleNamespace(
        means2d=np.zeros((n, 2)), conics=np.zeros((n, 3)), depths=np.zeros(n), colors=np.zeros((n, 3)),
        alphas=np.zeros(n), radii=np.zeros(n), ids=np.zeros(n, dtype=np.int64))
    st = OrStats()
    cam = make_camera(camera)
    m = lib().or_project(ca.n, _ptr(ca.pos), _ptr(ca.ls), _ptr(ca.rot), _ptr(ca.opac), _ptr(ca.sh), ca.K,
                         ctypes.byref(cam), _ptr(out.means2d), _ptr(out.conics), _ptr(out.depths),
                         _ptr(out.colors), _ptr(out.alphas), _ptr(out.radii), _ptr(out.ids), ctypes.byref(st))
    for k in ("means2d", "conics", "depths", "colors", "alphas", "radii", "ids"):
        setattr(out, k, getattr(out, k)[:m].copy())
    out.stats = st.as_dict()
    return out


def bin_tiles(means2d, radii, tiles_x, tiles_y):
    """renderer.py:80-101 -> (tile_starts int64[T+1], pair_splat int32[P])."""
    means2d = _f64(means2d)
    radii = _f64(radii)
    m = radii.shape[0]
    total = lib().or_count_pairs(m, _ptr(means2d), _ptr(radii), tiles_x, tiles_y)
    ts = np.zeros(tiles_x * tiles_y + 1, dtype=np.int64)
    ps = np.zeros(max(total, 1), dtype=np.int32)
    lib().or_bin_tiles(m, _ptr(means2d), _ptr(radii), tiles_x, tiles_y, _ptr(ts), _ptr(ps))
    return ts, ps[:total]


def blend(tiles_x, tile_size, width, height, tile_starts, pair_splat, means2d, conics, depths, colors, alphas):
    """_kernels_cy.blend_tile_range over all tiles on fresh accumulators (renderer.py:109-112).

    Returns (color_acc, alpha_acc, trans, depth_acc, contrib, visited).
    """
    ts = np.ascontiguousarray(tile_starts, dtype=np.int64)
    ps = np.ascontiguousarray(pair_splat, dtype=np.int32)
    arrs = [_f64(a) for a in (means2d, conics, depths, colors, alphas)]
    cacc = np.zeros((height, width, 3))
    aacc = np.zeros((height, width))
    tr = np.ones((height, width))
    dacc = np.zeros((height, width))
    contrib = np.zeros((height, width), dtype=np.int32)
    visited = np.zeros((height, width), dtype=np.int32)
    lib().or_blend(0, ts.size - 1, tiles_x, tile_size, width, height, _ptr(ts), _ptr(ps), *[_ptr(a) for a in arrs],
                   _ptr(cacc), _ptr(aacc), _ptr(tr), _ptr(dacc), _ptr(contrib), _ptr(visited))
    return cacc, aacc, tr, dacc, contrib, visited


def rasterize(cloud, camera, background, tiled=True, counters=True):
    """renderer.py:135 (tiled) / :145 (tiled=False). background None -> layer mode.

    Returns a namespace with color/alpha/depth (float64), contrib/visited (int32) and stats.
    """
    ca = _CloudArrays(cloud)
    h, w = int(camera.height), int(camera.width)
    cam = make_camera(camera, background)
    color = np.zeros((h, w, 3))
    alpha = np.zeros((h, w))
    depth = np.zeros((h, w))
    contrib = np.zeros((h, w), dtype=np.int32) if counters else None
    visited = np.zeros((h, w), dtype=np.int32) if counters else None
    st = OrStats()
    lib().or_rasterize(ctypes.byref(ca.c), ctypes.byref(cam), 1 if tiled else 0, 1 if background is None else 0,
                       _ptr(color), _ptr(alpha), _ptr(depth), _ptr(contrib), _ptr(visited), ctypes.byref(st))
    return SimpleNamespace(color=color, alpha=alpha, depth=depth, contrib=contrib, visited=visited,
                           stats=st.as_dict())


def rasterize_reference(cloud, camera, background, counters=True):
    return rasterize(cloud, camera, background, tiled=False, counters=counters)


def composite(front, back):
    """renderer.py:151-166 on float64 frames (namespaces/objects with color/alpha/depth)."""
    fc, fa, fd = _f64(front.color), _f64(front.alpha), _f64(front.depth)
    bc, ba, bd = _f64(back.color), _f64(back.alpha), _f64(back.depth)
    if fa.shape != ba.shape:
        raise ValueError(f"frame shapes differ: {fa.shape} vs {ba.shape}")
    oc, oa, od = np.empty_like(bc), np.empty_like(ba), np.empty_like(bd)
    lib().or_composite(fa.size, _ptr(fc), _ptr(fa), _ptr(fd), _ptr(bc), _ptr(ba), _ptr(bd), _ptr(oc), _ptr(oa),
                       _ptr(od))
    return SimpleNamespace(color=oc, alpha=oa, depth=od)


def concat_clouds(clouds):
    """cloud.py:110-129: concatenation with SH zero-padded to the largest K."""
    clouds = [c for c in clouds if np.asarray(c.positions).shape[0] > 0]
    if not clouds:
        return SimpleNamespace(positions=np.zeros((0, 3)), sh_coeffs=np.zeros((0, 1, 3)), opacities=np.zeros(0),
                               log_scales=np.zeros((0, 3)), rotations=np.zeros((0, 4)))
    k = max(np.asarray(c.sh_coeffs).shape[1] for c in clouds)
    sh = []
    for c in clouds:
        s = np.asarray(c.sh_coeffs, dtype=np.float64)
        if s.shape[1] < k:
            s = np.concatenate([s, np.zeros((s.shape[0], k - s.shape[1], 3))], axis=1)
        sh.append(s)
    cat = lambda name: np.concatenate([np.asarray(getattr(c, name), dtype=np.float64) for c in clouds])
    return SimpleNamespace(positions=cat("positions"), sh_coeffs=np.concatenate(sh), opacities=cat("opacities"),
                           log_scales=cat("log_scales"), rotations=cat("rotations"))


def render_observation(scene_cloud, avatar_clouds, camera, background):
    """renderer.py:169-177: scene pass + one concatenated avatar layer, depth-composited."""
    frame = rasterize(scene_cloud, camera, background)
    avatar_clouds = [c for c in avatar_clouds if np.asarray(c.positions).shape[0] > 0]
    if not avatar_clouds:
        return frame
    layer = rasterize(concat_clouds(avatar_clouds), camera, None)
    out = composite(layer, frame)
    out.scene, out.layer = frame, layer
    return out


def sample_pose(traj_quats, traj_trans, fps, t):
    """rig.py:78-104 on (T, J+1, 4)/(T, J+1, 3) arrays; returns (quats (J+1,4), trans (J+1,3))."""
    q = _f64(traj_quats)
    tr = _f64(traj_trans)
    nf, jp = q.shape[0], q.shape[1]
    oq = np.zeros((jp, 4))
    ot = np.zeros((jp, 3))
    rc = lib().or_sample_pose(nf, jp - 1, float(fps), _ptr(q), _ptr(tr), float(t), _ptr(oq), _ptr(ot))
    if rc != 0:
        raise ValueError(f"sample time must be nonnegative, got {t}")
    return oq, ot


def lbs_deform(positions, rotations, weights, inv_bind, pose_quats, pose_trans):
    """rig.py:107-146. pose_* include the root as the last row. Returns (positions, rotations) float64."""
    pos = _f64(positions)
    rot = _f64(rotations)
    w = _f64(weights)
    ib = _f64(inv_bind)
    pq = _f64(pose_quats)
    pt = _f64(pose_trans)
    n, j = w.shape
    op = np.zeros((n, 3))
    orr = np.zeros((n, 4))
    lib().or_lbs_deform(n, j, _ptr(pos), _ptr(rot), _ptr(w), _ptr(ib), _ptr(pq), _ptr(pt), _ptr(op), _ptr(orr))
    return op, orr


def render_batch(scene_cloud, avatar_clouds_per_env, cameras, background, threads=None):
    """E environments end to end (render_observation semantics) on `threads` host threads.

    avatar_clouds_per_env: list (len E) of already-deformed avatar clouds (concatenated per env)
    or None. Returns (color (E,H,W,3), alpha (E,H,W), depth (E,H,W)) float64.
    """
    if threads is None:
        threads = os.cpu_count() or 1
    e = len(cameras)
    h, w = int(cameras[0].height), int(cameras[0].width)
    sc = _CloudArrays(scene_cloud)
    keep = [sc]
    cams = (OrCamera * e)()
    for i, c in enumerate(cameras):
        cams[i] = make_camera(c, background)
    av = None
    if avatar_clouds_per_env is not None:
        av = (OrCloud * e)()
        for i, c in enumerate(avatar_clouds_per_env):
            if c is None:
                av[i] = OrCloud(0, 1, None, None, None, None, None)
            else:
                a = _CloudArrays(c)
                keep.append(a)
                av[i] = a.c
    color = np.zeros((e, h, w, 3))
    alpha = np.zeros((e, h, w))
    depth = np.zeros((e, h, w))
    lib().or_render_batch(ctypes.byref(sc.c), av, cams, e, int(threads), _ptr(color), _ptr(alpha), _ptr(depth))
    del keep
    return color, alpha, depth


def tiles_for(width, height):
    return math.ceil(width / TILE_SIZE), math.ceil(height / TILE_SIZE)


# ---------------------------------------------------------------------------------------------
# Asset loaders: numpy restatements of the reference's readers, used as the CPU
# baseline of scripts/bench_assets.py and as a second checker in tests. ply.py:76-120 +
# cloud.py:50-87 (float32 quaternion renormalization when any norm is off by more than 1e-5).

def load_gaussian_ply_numpy(path):
    """ply.load_gaussian_ply: returns (positions, sh (n,K,3), opacities, log_scales, rotations)."""
    with open(path, "rb") as f:
        props, n = [], None
        while True:
            line = f.readline().decode("ascii").strip()
            if line == "end_header":
                break
            parts = line.split()
            if parts and parts[0] == "element":
                if parts[1] == "vertex":
                    n = int(parts[2])
                    in_vertex = True
                else:
                    in_vertex = False
            elif parts and parts[0] == "property" and in_vertex:
                props.append(parts[2])
        data = f.read(n * len(props) * 4)
    table = np.frombuffer(data, dtype="<f4").reshape(n, len(props))
    col = {name: i for i, name in enumerate(props)}
    rest = sorted([p for p in props if p.startswith("f_rest_")], key=lambda s: int(s.rsplit("_", 1)[1]))
    k = (len(rest) // 3) + 1

    def cols(names):
        return table[:, [col[c] for c in names]]

    positions = cols(["x", "y", "z"]).copy()
    sh = np.zeros((n, k, 3), dtype=np.float32)
    sh[:, 0, :] = cols(["f_dc_0", "f_dc_1", "f_dc_2"])
    if rest:
        sh[:, 1:, :] = cols(rest).reshape(n, 3, k - 1).transpose(0, 2, 1)
    opacities = table[:, col["opacity"]].copy()
    log_scales = cols(["scale_0", "scale_1", "scale_2"]).copy()
    rotations = cols(["rot_0", "rot_1", "rot_2", "rot_3"]).copy()
    for a in (positions, sh, opacities, log_scales, rotations):
        if not np.isfinite(a).all():
            raise ValueError("non-finite values")
    norms = np.linalg.norm(rotations, axis=1)
    if (norms <= 0).any():
        raise ValueError("zero-norm rotation")
    if np.abs(norms - 1.0).max() > 1e-5:
        rotations = rotations / norms[:, None]
    return positions, sh, opacities, log_scales, rotations
