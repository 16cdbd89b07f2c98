"""Device-resident inputs for the CUDA path: packed clouds, avatar sets, camera structs.

Packing happens once per asset (scene load / bundle load), never per frame:
* DeviceCloud: (n,4) position+opacity, (n,4) log-scales, (n,4) wxyz rotations in float32 when the
  source arrays are float32 (the reference's cloud dtype) or float64 otherwise, so every value the
  float64 geometry reads is exactly the reference's; SH as a (K*3, n) float32
  structure-of-arrays so a warp's SH loads are coalesced.
* DeviceAvatars: A bundles concatenated in render_observation's concat order (cloud.py:110-129),
  canonical geometry in float64, skinning weights as up to 4 (joint, weight) influences per
  gaussian in ascending joint order (exactly the dense N x J rows, rig.py:119-132), trajectories
  and AvatarRuntime clock parameters (tasks.py:290-305).
"""

import numpy as np
import torch

from . import _native as N
from .errors import ContractViolation

MAX_INFLUENCES = 4


def _device(device):
    dev = torch.device(device if device is not None else "cuda")
    if dev.type != "cuda":
        raise ContractViolation(f"the splat renderer runs on CUDA devices only, got {dev}")
    return dev


def _pack4(a, width, dtype):
    a = np.asarray(a)
    out = np.zeros((a.shape[0], 4), dtype=dtype)
    out[:, :width] = a.reshape(a.shape[0], width)
    return out


def _sh_soa(sh, n):
    sh = np.asarray(sh)
    k = sh.shape[1] if sh.ndim == 3 else 1
    return np.ascontiguousarray(sh.reshape(n, k * 3).astype(np.float32).T), k


class DeviceCloud:
    """A GaussianCloud packed into the sn_cloud layout on a CUDA device."""

    def __init__(self, cloud, device=None):
        dev = _device(device)
        pos = np.asarray(cloud.positions)
        n = pos.shape[0]
        geo = [pos, cloud.opacities, cloud.log_scales, cloud.rotations]
        f32 = all(np.asarray(x).dtype == np.float32 for x in geo)
        dt = np.float32 if f32 else np.float64
        po = np.zeros((n, 4), dtype=dt)
        po[:, :3] = pos.reshape(n, 3)
        po[:, 3] = np.asarray(cloud.opacities).reshape(n)
        sh, k = _sh_soa(cloud.sh_coeffs, n)
        self.n = n
        self.sh_k = k
        self.dtype = N.SN_FLOAT32 if f32 else N.SN_FLOAT64
        self.device = dev
        self.pos_opacity = torch.from_numpy(po).to(dev)
        self.log_scales = torch.from_numpy(_pack4(cloud.log_scales, 3, dt)).to(dev)
        self.rotations = torch.from_numpy(_pack4(cloud.rotations, 4, dt)).to(dev)
        self.sh = torch.from_numpy(sh).to(dev)
        self.index = self.block_bounds = None
        self._struct = N.SnCloud(n, k, self.dtype, self.pos_opacity.data_ptr(), self.log_scales.data_ptr(),
                                 self.rotations.data_ptr(), self.sh.data_ptr(), None, None)

    @classmethod
    def wrap(cls, cloud, device=None):
        return cloud if isinstance(cloud, DeviceCloud) else cls(cloud, device)

    @classmethod
    def from_device(cls, pos_opacity, log_scales, rotations, sh, sh_k, dtype, device):
        """Wrap buffers already in the sn_cloud layout (e.g. unpacked by assets.load_gaussian_ply)."""
        self = cls.__new__(cls)
        self.n = int(pos_opacity.shape[0])
        self.sh_k = int(sh_k)
        self.dtype = dtype
        self.device = device
        self.pos_opacity, self.log_scales, self.rotations, self.sh = pos_opacity, log_scales, rotations, sh
        self.index = self.block_bounds = None
        self._struct = N.SnCloud(self.n, self.sh_k, dtype, pos_opacity.data_ptr(), log_scales.data_ptr(),
                                 rotations.data_ptr(), sh.data_ptr(), None, None)
        return self

    def spatially_ordered(self):
        """A copy with the rows in Morton (Z-curve) order of the positions, carrying each row's
        original index and the bounding box of every 256-row block (sn_cloud ABI 3): the count
        kernel decides whole blocks per env where the box allows, and every order-dependent output
        (depth ties, ids) uses the original index, so renders equal the original order's."""
        if self.index is not None:
            return self
        pos = self.pos_opacity[:, :3].double()
        n = self.n
        lo = pos.amin(0) if n else torch.zeros(3, dtype=torch.float64, device=pos.device)
        hi = pos.amax(0) if n else lo
        span = (hi - lo).clamp_min(1e-30)
        q = ((pos - lo) / span * 1023.0).clamp(0, 1023).long()

        def spread(v):  # 10 bits -> every third bit
            v = (v | (v << 16)) & 0x030000FF
            v = (v | (v << 8)) & 0x0300F00F
            v = (v | (v << 4)) & 0x030C30C3
            return (v | (v << 2)) & 0x09249249

        code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
        perm = torch.sort(code, stable=True).indices
        out = DeviceCloud.__new__(DeviceCloud)
        out.n, out.sh_k, out.dtype, out.device = n, self.sh_k, self.dtype, self.device
        out.pos_opacity = self.pos_opacity[perm].contiguous()
        out.log_scales = self.log_scales[perm].contiguous()
        out.rotations = self.rotations[perm].contiguous()
        out.sh = self.sh[:, perm].contiguous()
        out.index = perm.to(torch.int32).contiguous()
        nb = (n + 255) // 256
        p = out.pos_opacity[:, :3].double()
        pmin = torch.full((nb * 256, 3), float("inf"), dtype=torch.float64, device=p.device)
        pmax = torch.full((nb * 256, 3), float("-inf"), dtype=torch.float64, device=p.device)
        pmin[:n] = p
        pmax[:n] = p
        bmin = pmin.view(nb, 256, 3).amin(1)
        bmax = pmax.view(nb, 256, 3).amax(1)
        # float32 bounds rounded outward (exact for float32 positions)
        lo32, hi32 = bmin.float(), bmax.float()
        lo32 = torch.where(lo32.double() > bmin, torch.nextafter(lo32, torch.full_like(lo32, -float("inf"))), lo32)
        hi32 = torch.where(hi32.double() < bmax, torch.nextafter(hi32, torch.full_like(hi32, float("inf"))), hi32)
        out.block_bounds = torch.cat([lo32, hi32, torch.zeros(nb, 2, dtype=torch.float32, device=p.device)],
                                     dim=1).contiguous()
        out._struct = N.SnCloud(n, out.sh_k, out.dtype, out.pos_opacity.data_ptr(), out.log_scales.data_ptr(),
                                out.rotations.data_ptr(), out.sh.data_ptr(), out.index.data_ptr(),
                                out.block_bounds.data_ptr())
        return out

    def to_host(self):
        """(positions (n,3), sh_coeffs (n,K,3), opacities (n,), log_scales (n,3), rotations (n,4)), in
        the original row order"""
        po = self.pos_opacity.cpu().numpy()
        sh = self.sh.cpu().numpy().T.reshape(self.n, self.sh_k, 3)
        ls, rot = self.log_scales.cpu().numpy()[:, :3], self.rotations.cpu().numpy()
        if self.index is not None:
            inv = np.empty(self.n, dtype=np.int64)
            inv[self.index.cpu().numpy()] = np.arange(self.n)
            po, sh, ls, rot = po[inv], sh[inv], ls[inv], rot[inv]
        return po[:, :3], sh, po[:, 3], ls, rot

    def struct(self):
        return self._struct


def influence_widths(weights):
    """Nonzero influences per row of dense (N, J) skinning weights."""
    return (np.asarray(weights) != 0.0).sum(axis=1)


def sparse_influences(weights, max_influences=MAX_INFLUENCES):
    """Dense (N, J) skinning weights -> (joints uint32 packed 4 x uint8, weights (N, 4) float64),
    the 4-slot layout for rows with at most 4 nonzeros (csr_influences takes any width).

    Influences are the nonzero entries of each row in ascending joint order, so the kernel's
    running sums visit joints in the same order as the reference's dense contractions.
    """
    w = np.asarray(weights, dtype=np.float64)
    n, j = w.shape
    if j > 255:
        raise ContractViolation(f"at most 255 joints are supported, got {j}")
    nz = w != 0.0
    counts = nz.sum(axis=1)
    if n and counts.max() > max_influences:
        row = int(np.argmax(counts))
        raise ContractViolation(f"weight row {row} has {int(counts[row])} nonzero joints; the 4-slot layout "
                                f"holds at most {max_influences} (use csr_influences)")
    order = np.argsort(~nz, axis=1, kind="stable")[:, :max_influences]  # nonzeros first, ascending joint
    wk = np.take_along_axis(w, order, axis=1)
    slot_used = np.arange(max_influences)[None, :] < counts[:, None]
    wk = np.where(slot_used, wk, 0.0)
    jk = np.where(slot_used, order, 0).astype(np.uint32)
    if max_influences < 4:
        pad = 4 - max_influences
        wk = np.pad(wk, ((0, 0), (0, pad)))
        jk = np.pad(jk, ((0, 0), (0, pad)))
    packed = jk[:, 0] | (jk[:, 1] << 8) | (jk[:, 2] << 16) | (jk[:, 3] << 24)
    return packed.astype(np.uint32), np.ascontiguousarray(wk)


def csr_influences(weights, row_offset=0):
    """Dense (N, J) skinning weights -> CSR (offsets uint32 (N+1), joints uint8 (nnz), weights f64
    (nnz)): each row's nonzeros in ascending joint order, any width (dense SMPL / SMPL-X skins).
    `row_offset` is added to every offset (concatenating several bundles)."""
    w = np.asarray(weights, dtype=np.float64)
    n, j = w.shape
    if j > 255:
        raise ContractViolation(f"at most 255 joints are supported, got {j}")
    rows, cols = np.nonzero(w)  # row-major: ascending joint within each row
    counts = np.bincount(rows, minlength=n)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    off += row_offset
    if off[-1] >= 2 ** 32:
        raise ContractViolation("too many skinning influences for 32-bit offsets")
    return off.astype(np.uint32), cols.astype(np.uint8), np.ascontiguousarray(w[rows, cols])


class DeviceAvatars:
    """A set of avatar bundles (+ AvatarRuntime clocking) packed into the sn_avatars layout.

    bundles: AvatarBundle-like objects (.canonical, .lbs_weights, .inv_bind, .trajectory).
    start_offsets / loops: per avatar (AvatarRuntime.start_offset / .loop).
    """

    def __init__(self, bundles, start_offsets=None, loops=None, device=None):
        dev = _device(device)
        bundles = list(bundles)
        if not bundles:
            raise ContractViolation("need at least one avatar bundle")
        a = len(bundles)
        joints = {int(np.asarray(b.lbs_weights).shape[1]) for b in bundles}
        if len(joints) != 1:
            raise ContractViolation(f"all avatars of a set must share the joint count, got {sorted(joints)}")
        j = joints.pop()
        k = max(np.asarray(b.canonical.sh_coeffs).shape[1] for b in bundles)
        counts = [int(np.asarray(b.canonical.positions).shape[0]) for b in bundles]
        n = sum(counts)
        self.offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        po = np.zeros((n, 4))
        ls = np.zeros((n, 4))
        rot = np.zeros((n, 4))
        sh = np.zeros((n, k, 3), dtype=np.float32)
        # 4-slot influences when every row has <= 4 nonzeros, else CSR rows for the whole set
        csr = any(n_b and influence_widths(b.lbs_weights).max() > MAX_INFLUENCES
                  for n_b, b in zip(counts, bundles))
        jpk = np.zeros(n, dtype=np.uint32)
        wts = np.zeros((n, 4))
        c_off, c_j, c_w = [np.zeros(1, dtype=np.uint32)], [], []
        owner = np.zeros(n, dtype=np.uint16)
        ib = np.zeros((a, j, 16))
        tq, tt, toff, nf, fps = [], [], [], [], []
        frame_off = 0
        for i, b in enumerate(bundles):
            s, e = self.offsets[i], self.offsets[i + 1]
            c = b.canonical
            po[s:e, :3] = np.asarray(c.positions, dtype=np.float64)
            po[s:e, 3] = np.asarray(c.opacities, dtype=np.float64)
            ls[s:e, :3] = np.asarray(c.log_scales, dtype=np.float64)
            rot[s:e] = np.asarray(c.rotations, dtype=np.float64)
            cs = np.asarray(c.sh_coeffs, dtype=np.float32)
            sh[s:e, :cs.shape[1]] = cs
            if csr:
                o, jj, ww = csr_influences(b.lbs_weights, row_offset=int(c_off[-1][-1]))
                c_off.append(o[1:])
                c_j.append(jj)
                c_w.append(ww)
            else:
                jpk[s:e], wts[s:e] = sparse_influences(b.lbs_weights)
            owner[s:e] = i
            ib[i] = np.asarray(b.inv_bind, dtype=np.float64).reshape(j, 16)
            traj = b.trajectory
            q = np.asarray(traj.quats, dtype=np.float64)
            if q.shape[1] != j + 1:
                raise ContractViolation(f"trajectory of avatar {i} has {q.shape[1] - 1} joints, weights have {j}")
            tq.append(q.reshape(-1))
            tt.append(np.asarray(traj.trans, dtype=np.float64).reshape(-1))
            toff.append(frame_off)
            nf.append(q.shape[0])
            fps.append(float(traj.fps))
            frame_off += q.shape[0]
        t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        infl = None
        if csr:
            cj, cw = np.concatenate(c_j), np.concatenate(c_w)
            # (one padding entry keeps the buffers non-null for an all-zero skin)
            infl = (t(np.concatenate(c_off).view(np.int32)), t(np.concatenate([cj, np.zeros(1, np.uint8)])),
                    t(np.concatenate([cw, np.zeros(1)])))
        self._finish(t(po), t(ls), t(rot), t(sh.reshape(n, k * 3).T), t(jpk.view(np.int32)), t(wts), counts, ib,
                     tq, tt, toff, nf, fps, j, k, start_offsets, loops, dev, infl)

    @classmethod
    def from_device(cls, po, ls, rot, sh, joints, weights, counts, specs, j, k, start_offsets, loops, device,
                    infl=None):
        """Canonical buffers already on the device (assets.load_avatar_bundles); specs carry each
        bundle's inv_bind and trajectory (host, float64); infl = (offsets, joints, weights) CSR
        device tensors for skins wider than 4 influences."""
        self = cls.__new__(cls)
        ib = np.stack([np.asarray(s.inv_bind, dtype=np.float64).reshape(j, 16) for s in specs])
        tq, tt, toff, nf, fps = [], [], [], [], []
        frame_off = 0
        for s in specs:
            q = np.asarray(s.trajectory.quats, dtype=np.float64)
            tq.append(q.reshape(-1))
            tt.append(np.asarray(s.trajectory.trans, dtype=np.float64).reshape(-1))
            toff.append(frame_off)
            nf.append(q.shape[0])
            fps.append(float(s.trajectory.fps))
            frame_off += q.shape[0]
        self._finish(po, ls, rot, sh, joints, weights, counts, ib, tq, tt, toff, nf, fps, j, k, start_offsets, loops,
                     device, infl)
        return self

    def _finish(self, po, ls, rot, sh, joints, weights, counts, ib, tq, tt, toff, nf, fps, j, k, start_offsets, loops,
                dev, infl=None):
        a = len(counts)
        n = int(sum(counts))
        self.offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        owner = np.repeat(np.arange(a, dtype=np.uint16), counts)
        so = np.zeros(a) if start_offsets is None else np.asarray(start_offsets, dtype=np.float64)
        lp = np.ones(a, dtype=np.int32) if loops is None else np.asarray(loops, dtype=np.int32)
        t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
        self.n, self.n_avatars, self.n_joints, self.sh_k, self.device = n, a, j, k, dev
        self.counts = list(counts)
        self.pos_opacity, self.log_scales, self.rotations, self.sh = po, ls, rot, sh
        self.joints, self.weights, self.avatar_of = joints, weights, t(owner.view(np.int16))
        self.inv_bind = t(ib)
        self.traj_q, self.traj_t = t(np.concatenate(tq)), t(np.concatenate(tt))
        self.traj_offset = t(np.asarray(toff, dtype=np.int64))
        self.n_frames = t(np.asarray(nf, dtype=np.int32))
        self.fps = t(np.asarray(fps, dtype=np.float64))
        self.start_offset = t(so)
        self.loop = t(lp)
        self.infl = infl  # CSR (offsets, joints, weights) or None (4-slot layout)
        ptr = lambda x: x.data_ptr()
        iptr = (None, None, None) if infl is None else tuple(x.data_ptr() for x in infl)
        self._struct = N.SnAvatars(
            n, a, j, k, 0, ptr(self.pos_opacity), ptr(self.log_scales), ptr(self.rotations), ptr(self.sh),
            ptr(self.joints), ptr(self.weights), ptr(self.avatar_of), ptr(self.inv_bind), ptr(self.traj_q),
            ptr(self.traj_t), ptr(self.traj_offset), ptr(self.n_frames), ptr(self.fps), ptr(self.start_offset),
            ptr(self.loop), *iptr)

    def struct(self):
        return self._struct


CAMERA_DTYPE = np.dtype([("intr", "<f8", 6), ("rot", "<f8", 9), ("trans", "<f8", 3), ("center", "<f8", 3),
                         ("background", "<f8", 3), ("size", "<i4", 2), ("has_background", "<i4"), ("pad", "<i4")])
assert CAMERA_DTYPE.itemsize == 208


def camera_array(cameras, background):
    """Cameras -> ctypes array of sn_camera (host). `center` is evaluated exactly as the reference's
    Camera.center (camera.py:43-48): -R^T @ t with numpy."""
    e = len(cameras)
    arr = np.zeros(e, dtype=CAMERA_DTYPE)
    for i, c in enumerate(cameras):
        w2c = np.asarray(c.world_to_camera, dtype=np.float64)
        r = w2c[:3, :3]
        t = w2c[:3, 3]
        arr[i]["intr"] = (c.fx, c.fy, c.cx, c.cy, c.near, c.far)
        arr[i]["rot"] = r.reshape(9)
        arr[i]["trans"] = t
        arr[i]["center"] = -r.T @ t
        arr[i]["size"] = (int(c.width), int(c.height))
    if background is None:
        arr["has_background"] = 0
    else:
        bg = np.asarray(background, dtype=np.float64)
        arr["background"] = bg.reshape(-1, 3) if bg.ndim == 2 else bg[None, :]
        arr["has_background"] = 1
    buf = (N.SnCamera * e)()
    ctypes_bytes = np.frombuffer(buf, dtype=np.uint8)
    ctypes_bytes[:] = arr.view(np.uint8)
    return buf
