"""Asset ingest straight to the device.

* load_gaussian_ply(path) -> DeviceCloud: the reference's PLY reader (splatnav/ply.py:18-120:
  header grammar, errors, f_rest channel-major on disk) with the float32 vertex payload uploaded as
  is and unpacked by a CUDA kernel (sn_unpack_ply) into the renderer's layout, including
  GaussianCloud.validate (cloud.py:50-87): non-finite checks and the float32 quaternion
  renormalization, bit-for-bit.
* load_avatar_bundles(paths) -> DeviceAvatars: the reference's bundle directory reader
  (splatnav/avatar.py:180-254: manifest schema, blob sizes, capsules) with canonical.f32 and
  weights.f32 unpacked on the device (sn_unpack_bundle): float64 canonical geometry, SH SoA, the
  dense N x J weights -> each row's nonzero (joint, weight) influences (4-slot, or CSR for wider
  skins) with AvatarBundle.validate's checks and float64 row renormalization in numpy's summation
  order; trajectory, inverse-bind and capsule-track checks on the host.

Both raise the reference's exception types with the reference's messages.
"""

import ctypes
import json
import os

import numpy as np
import torch

from . import _native as N
from .avatar import CapsuleTrack, Skeleton, Trajectory
from .device import DeviceAvatars, DeviceCloud, _device
from .errors import (ConsistencyError, ContractViolation, PlyParseError, SchemaError, UnsupportedLayoutError,
                     ValidationError)

_REST_COUNT_TO_DEGREE = {0: 0, 9: 1, 24: 2, 45: 3}
_FIELDS = ("positions", "sh_coeffs", "opacities", "log_scales", "rotations")
_MANIFEST_KEYS = ("n_gaussians", "n_joints", "sh_degree", "fps", "n_frames", "n_capsules", "skeleton")
WEIGHT_RENORM_TOL = 1e-3


# ------------------------------------------------------------------------------------------ PLY

def _read_header(f):
    """ply.py:18-30"""
    lines = []
    while True:
        raw = f.readline()
        if not raw:
            raise PlyParseError("unexpected end of file before 'end_header'")
        try:
            line = raw.decode("ascii").strip()
        except UnicodeDecodeError:
            raise PlyParseError(f"non-ascii bytes in header line {len(lines) + 1}") from None
        lines.append(line)
        if line == "end_header":
            return lines


def _parse_header(lines):
    """ply.py:33-73"""
    if not lines or lines[0] != "ply":
        raise PlyParseError(f"first header line is {lines[0]!r}, expected 'ply'")
    fmt = lines[1] if len(lines) > 1 else ""
    if fmt != "format binary_little_endian 1.0":
        raise PlyParseError(f"unsupported format line {fmt!r}; only binary_little_endian 1.0 is handled")
    n_vertices = None
    properties = []
    in_vertex = False
    for line in lines[2:]:
        if line.startswith("comment") or line == "end_header" or not line:
            continue
        parts = line.split()
        if parts[0] == "element":
            if parts[1] == "vertex":
                if len(parts) != 3:
                    raise PlyParseError(f"malformed element line {line!r}")
                try:
                    n_vertices = int(parts[2])
                except ValueError:
                    raise PlyParseError(f"bad vertex count in line {line!r}") from None
                in_vertex = True
            elif n_vertices is None:
                raise PlyParseError(f"element {parts[1]!r} precedes the vertex element; cannot locate payload")
            else:
                in_vertex = False
        elif parts[0] == "property":
            if not in_vertex:
                continue
            if len(parts) != 3:
                raise PlyParseError(f"malformed property line {line!r}")
            ptype, pname = parts[1], parts[2]
            if ptype not in ("float", "float32"):
                raise PlyParseError(f"property {pname!r} has type {ptype!r}; only float32 is handled")
            properties.append(pname)
        else:
            raise PlyParseError(f"unrecognized header line {line!r}")
    if n_vertices is None:
        raise PlyParseError("header declares no vertex element")
    return n_vertices, properties


def read_ply_table(path, pinned=False):
    """Header + the raw vertex payload as a (n, n_props) float32 array (read straight into pinned
    host memory when `pinned`, ready for the upload); the column indices the unpack kernel reads
    (x y z f_dc_0..2 opacity scale_0..2 rot_0..3 f_rest_0..) and K."""
    with open(path, "rb") as f:
        lines = _read_header(f)
        n, props = _parse_header(lines)
        nbytes = n * len(props) * 4
        buf = torch.empty(nbytes, dtype=torch.uint8, pin_memory=pinned and nbytes > 0)
        got = f.readinto(memoryview(buf.numpy())) if nbytes else 0
    if got != nbytes:
        raise PlyParseError(f"payload truncated: expected {nbytes} bytes, got {got}")
    data = buf.numpy()
    col = {name: i for i, name in enumerate(props)}
    required = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity",
                "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    missing = [r for r in required if r not in col]
    if missing:
        raise UnsupportedLayoutError(f"missing required properties: {missing}")
    rest_names = [p for p in props if p.startswith("f_rest_")]
    n_rest = len(rest_names)
    if n_rest not in _REST_COUNT_TO_DEGREE:
        raise UnsupportedLayoutError(
            f"{n_rest} f_rest properties match no SH degree; expected one of {sorted(_REST_COUNT_TO_DEGREE)}")
    expected = [f"f_rest_{i}" for i in range(n_rest)]
    if sorted(rest_names, key=lambda s: int(s.rsplit("_", 1)[1])) != expected:
        raise UnsupportedLayoutError("f_rest properties are not a contiguous 0-based sequence")
    k = (_REST_COUNT_TO_DEGREE[n_rest] + 1) ** 2
    cols = np.array([col[c] for c in required[:6]] + [col["opacity"]] + [col[c] for c in required[7:]] +
                    [col[c] for c in expected], dtype=np.int32)
    table = data.view("<f4").reshape(n, len(props)) if props else np.zeros((n, 0), "<f4")
    return table, cols, k


def _raise_cloud_errors(flags_dev, counters):
    """GaussianCloud.validate's messages (cloud.py:66-83) from the kernel's counters and flags."""
    if any(counters[i] for i in range(6)):
        flags = flags_dev.cpu().numpy()
        for b, name in enumerate(_FIELDS):
            if counters[b]:
                idx = np.nonzero(flags & (1 << b))[0]
                head = ", ".join(str(i) for i in idx[:10])
                more = "..." if idx.size > 10 else ""
                raise ValidationError(f"non-finite values in {name} at splat indices [{head}{more}]")
        idx = np.nonzero(flags & 32)[0]
        raise ValidationError(f"zero-norm rotation quaternions at indices {idx[:10].tolist()}")


def load_gaussian_ply(path, device=None, stream=None):
    """ply.load_gaussian_ply (ply.py:76-120) straight into a DeviceCloud."""
    dev = _device(device)
    table, cols, k = read_ply_table(path, pinned=True)
    n = table.shape[0]
    t = torch.from_numpy(table).to(dev, non_blocking=True)
    pos = torch.empty((n, 4), dtype=torch.float32, device=dev)
    ls = torch.empty((n, 4), dtype=torch.float32, device=dev)
    rot = torch.empty((n, 4), dtype=torch.float32, device=dev)
    sh = torch.empty((k * 3, n), dtype=torch.float32, device=dev)
    flags = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(10, dtype=torch.int64, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    lib = N.load()
    N.check(lib.sn_unpack_ply(n, table.shape[1], t.data_ptr(), cols.ctypes.data_as(ctypes.c_void_p), k,
                              pos.data_ptr(), ls.data_ptr(), rot.data_ptr(), sh.data_ptr(), flags.data_ptr(),
                              cnt.data_ptr(), st.cuda_stream))
    counters = cnt.cpu().numpy().view(np.uint64)
    _raise_cloud_errors(flags, counters)
    return DeviceCloud.from_device(pos, ls, rot, sh, k, N.SN_FLOAT32, dev)


# --------------------------------------------------------------------------------- avatar bundles

def _read_blob(dirpath, name, count):
    """avatar.py:180-188"""
    path = os.path.join(dirpath, name)
    if not os.path.isfile(path):
        raise FileNotFoundError(f"avatar bundle is missing blob '{name}' in {dirpath}")
    data = np.fromfile(path, dtype="<f4")
    if data.size != count:
        raise ConsistencyError(f"blob '{name}' holds {data.size} floats, manifest implies {count}")
    return data


def read_bundle_dir(path, require_capsules=True):
    """The host part of load_avatar_bundle (avatar.py:191-254): manifest, blobs, skeleton and
    trajectory (validated); canonical.f32 and weights.f32 stay raw float32 for the device."""
    manifest_path = os.path.join(path, "manifest.json")
    if not os.path.isfile(manifest_path):
        raise FileNotFoundError(f"avatar bundle is missing manifest.json in {path}")
    with open(manifest_path, "r", encoding="utf-8") as f:
        manifest = json.load(f)
    missing = [key for key in _MANIFEST_KEYS if key not in manifest]
    if missing:
        raise SchemaError(f"manifest.json missing keys: {missing}")
    n = int(manifest["n_gaussians"])
    j = int(manifest["n_joints"])
    degree = int(manifest["sh_degree"])
    fps = float(manifest["fps"])
    t = int(manifest["n_frames"])
    c = int(manifest["n_capsules"])
    if not 0 <= degree <= 3:
        raise ValidationError(f"sh_degree must be 0..3, got {degree}")
    k = (degree + 1) ** 2
    skel_entries = manifest["skeleton"]
    if len(skel_entries) != j:
        raise SchemaError(f"manifest skeleton lists {len(skel_entries)} joints, n_joints is {j}")
    parents = np.array([entry["parent"] for entry in skel_entries], dtype=np.int64)
    rest_pos = np.array([entry["rest_pos"] for entry in skel_entries], dtype=np.float64)
    skeleton = Skeleton(parents, rest_pos)
    floats_per_splat = 3 + 3 + 3 * (k - 1) + 1 + 3 + 4
    canonical = _read_blob(path, "canonical.f32", n * floats_per_splat)
    weights = _read_blob(path, "weights.f32", n * j)
    inv_bind = _read_blob(path, "inv_bind.f32", j * 16).reshape(j, 4, 4).astype(np.float64)
    traj_raw = _read_blob(path, "trajectory.f32", t * (j + 1) * 7).reshape(t, j + 1, 7).astype(np.float64)
    trajectory = Trajectory(fps=fps, quats=traj_raw[:, :, :4], trans=traj_raw[:, :, 4:])
    capsules = None
    if os.path.isfile(os.path.join(path, "capsules.f32")):
        capsules = CapsuleTrack(_read_blob(path, "capsules.f32", t * c * 7).reshape(t, c, 7).astype(np.float64))
    elif require_capsules:
        raise FileNotFoundError(f"avatar bundle is missing blob 'capsules.f32' in {path}")
    # validated by load_avatar_bundles in AvatarBundle.validate's order (canonical cloud first)
    return {"n": n, "j": j, "k": k, "canonical": canonical, "weights": weights, "inv_bind": inv_bind,
            "trajectory": trajectory, "skeleton": skeleton, "capsules": capsules}


def _validate_host_parts(s):
    """AvatarBundle.validate (avatar.py:155-178) for everything but the canonical cloud and the
    weights (checked on the device): skeleton, trajectory (incl. non-finite data), shapes,
    non-finite inverse binds. The capsule track is checked after the weights (_validate_capsules)."""
    j = s["j"]
    s["skeleton"].validate()
    s["trajectory"].validate()
    if s["inv_bind"].shape != (j, 4, 4):
        raise ConsistencyError(f"inv_bind shape {s['inv_bind'].shape} != ({j}, 4, 4)")
    if s["trajectory"].n_joints != j:
        raise ConsistencyError(f"trajectory has {s['trajectory'].n_joints} joints, skeleton has {j}")
    if not np.isfinite(s["inv_bind"]).all():
        raise ValidationError("non-finite inverse bind matrices")


def _validate_capsules(s):
    cap = s["capsules"]
    if cap is None:
        return
    cap.validate()
    if cap.n_frames != s["trajectory"].n_frames:
        raise ConsistencyError(f"capsule track has {cap.n_frames} frames, trajectory has {s['trajectory'].n_frames}")


class _BundleSpec:
    """What DeviceAvatars reads from a bundle besides the canonical cloud and the weights."""

    def __init__(self, d):
        self.n_gaussians, self.sh_k = d["n"], d["k"]
        self.inv_bind, self.trajectory = d["inv_bind"], d["trajectory"]


def load_avatar_bundles(paths, start_offsets=None, loops=None, device=None, require_capsules=True):
    """load_avatar_bundle for each directory, packed into one DeviceAvatars (concat order) with the
    canonical clouds and skinning weights unpacked and validated on the device."""
    dev = _device(device)
    specs = [read_bundle_dir(p, require_capsules) for p in paths]
    if not specs:
        raise ContractViolation("need at least one avatar bundle")
    joints = {s["j"] for s in specs}
    if len(joints) != 1:
        raise ContractViolation(f"all avatars of a set must share the joint count, got {sorted(joints)}")
    j = joints.pop()
    k = max(s["k"] for s in specs)
    counts = [s["n"] for s in specs]
    n = sum(counts)
    # skins with a row wider than 4 nonzero influences use the CSR layout for the whole set (row
    # offsets counted here from the raw float32 rows; joints and weights are packed on the device)
    widths = [(s["weights"].reshape(s["n"], j) != 0.0).sum(axis=1) for s in specs]
    csr = any(w.size and int(w.max()) > 4 for w in widths)
    po = torch.zeros((n, 4), dtype=torch.float64, device=dev)
    ls = torch.zeros((n, 4), dtype=torch.float64, device=dev)
    rot = torch.zeros((n, 4), dtype=torch.float64, device=dev)
    sh = torch.zeros((k * 3, n), dtype=torch.float32, device=dev)
    jpk = torch.zeros(n, dtype=torch.int32, device=dev)
    wts = torch.zeros((n, 4), dtype=torch.float64, device=dev)
    infl = None
    if csr:
        off = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.concatenate(widths), out=off[1:])
        if off[-1] >= 2 ** 32:
            raise ContractViolation("too many skinning influences for 32-bit offsets")
        nnz = int(off[-1])
        infl = (torch.from_numpy(off.astype(np.uint32).view(np.int32)).to(dev),
                torch.zeros(nnz + 1, dtype=torch.uint8, device=dev), torch.zeros(nnz + 1, dtype=torch.float64, device=dev))
    st = torch.cuda.current_stream(dev)
    lib = N.load()
    row0 = 0
    for path, s in zip(paths, specs):
        m = s["n"]
        canon = torch.from_numpy(s["canonical"]).to(dev)
        w = torch.from_numpy(s["weights"]).to(dev)
        sums = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
        flags = torch.zeros(max(m, 1), dtype=torch.uint8, device=dev)
        cnt = torch.zeros(10, dtype=torch.int64, device=dev)
        N.check(lib.sn_unpack_bundle(m, s["k"], j, canon.data_ptr(), w.data_ptr(), row0, n, po.data_ptr(),
                                     ls.data_ptr(), rot.data_ptr(), sh.data_ptr(), jpk.data_ptr(), wts.data_ptr(),
                                     sums.data_ptr(), flags.data_ptr(), cnt.data_ptr(), st.cuda_stream))
        if csr:
            N.check(lib.sn_pack_influences(m, j, w.data_ptr(), sums.data_ptr(), cnt.data_ptr(),
                                           infl[0].data_ptr() + 4 * row0, infl[1].data_ptr(), infl[2].data_ptr(),
                                           st.cuda_stream))
        counters = cnt.cpu().numpy().view(np.uint64)
        _raise_cloud_errors(flags, counters)                      # AvatarBundle.validate: canonical first
        _validate_host_parts(s)
        if m:
            if counters[7]:
                raise ValidationError("negative skinning weights")
            max_dev = float(np.uint64(counters[9]).view(np.float64))
            if max_dev > WEIGHT_RENORM_TOL:
                dev_rows = np.abs(sums.cpu().numpy()[:m] - 1.0)
                bad = int(np.argmax(dev_rows))
                raise ValidationError(f"weight row {bad} sums to {sums[bad].item():.6f}; deviation exceeds "
                                      f"{WEIGHT_RENORM_TOL}")
        _validate_capsules(s)
        row0 += m
    return DeviceAvatars.from_device(po, ls, rot, sh, jpk, wts, counts, [_BundleSpec(s) for s in specs], j, k,
                                     start_offsets, loops, dev, infl)
