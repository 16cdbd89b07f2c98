"""Drop-in avatar rig entry points (reference: splatnav/rig.py:36-146, tasks.py:290-320).

sample_pose and lbs_deform keep the reference signatures and return types (JointPose,
GaussianCloud with float64 positions/rotations) but run on the GPU: the pose kernel
(csrc/sn_rig.cu) and the skinning kernel (csrc/sn_preprocess.cu, the same device code the fused
render path uses). For rendering many environments, prefer batch.BatchRenderer, which never
materializes deformed clouds: skinning is fused into the avatar-layer projection.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .cloud import GaussianCloud
from .device import DeviceAvatars
from .errors import ContractViolation


@dataclass
class JointPose:
    """World joint transforms (J,4) quats + (J,3) translations, plus a root transform."""

    quats: np.ndarray
    trans: np.ndarray
    root_quat: np.ndarray
    root_trans: np.ndarray

    @property
    def n_joints(self):
        return self.quats.shape[0]


class _TrajectoryOnly:
    """Minimal sn_avatars view holding one trajectory (for sample_pose)."""

    def __init__(self, trajectory, dev):
        q = np.ascontiguousarray(np.asarray(trajectory.quats, dtype=np.float64))
        t = np.ascontiguousarray(np.asarray(trajectory.trans, dtype=np.float64))
        self.jp = q.shape[1]
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self.tensors = [to(q.reshape(-1)), to(t.reshape(-1)), to(np.zeros(1, dtype=np.int64)),
                        to(np.array([q.shape[0]], dtype=np.int32)), to(np.array([float(trajectory.fps)])),
                        to(np.zeros(1)), to(np.zeros(1, dtype=np.int32)), to(np.zeros((1, self.jp - 1, 16)))]
        tq, tt, toff, nf, fps, so, lp, ib = [x.data_ptr() for x in self.tensors]
        self.s = N.SnAvatars(0, 1, self.jp - 1, 1, 0, None, None, None, None, None, None, None, ib, tq, tt, toff, nf,
                             fps, so, lp)


def sample_pose(trajectory, t):
    """rig.py:78-104: interpolate joint transforms at time t (seconds); clamps past the end."""
    if t < 0:
        raise ContractViolation(f"sample time must be nonnegative, got {t}")
    dev = torch.device("cuda")
    view = _TrajectoryOnly(trajectory, dev)
    jp = view.jp
    pq = torch.empty((jp, 4), dtype=torch.float64, device=dev)
    pt = torch.empty((jp, 3), dtype=torch.float64, device=dev)
    times = np.array([float(t)])
    stream = torch.cuda.current_stream(dev).cuda_stream
    lib = N.load()
    N.check(lib.sn_sample_pose(N.default_context().handle, ctypes.byref(view.s), times.ctypes.data_as(ctypes.c_void_p),
                               1, pq.data_ptr(), pt.data_ptr(), stream))
    q = pq.cpu().numpy()
    tr = pt.cpu().numpy()
    return JointPose(quats=q[:-1].copy(), trans=tr[:-1].copy(), root_quat=q[-1].copy(), root_trans=tr[-1].copy())


def skin_device(dev_avatars, avatar, pose_q, pose_t, context=None):
    """Skin avatar `avatar` of a DeviceAvatars set at device poses (J+1,4)/(J+1,3) -> device
    float64 positions (n,3), rotations (n,4)."""
    lib = N.load()
    ctx = context or N.default_context()
    g0 = int(dev_avatars.offsets[avatar])
    n = int(dev_avatars.offsets[avatar + 1]) - g0
    dev = dev_avatars.device
    pos = torch.empty((n, 3), dtype=torch.float64, device=dev)
    rot = torch.empty((n, 4), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check(lib.sn_skin_lbs(ctx.handle, ctypes.byref(dev_avatars.struct()), avatar, g0, n, pose_q.data_ptr(),
                            pose_t.data_ptr(), pos.data_ptr(), rot.data_ptr(), stream))
    return pos, rot


def pose_tensors(pose, device):
    q = np.concatenate([np.asarray(pose.quats, dtype=np.float64), np.asarray(pose.root_quat, dtype=np.float64)[None]])
    t = np.concatenate([np.asarray(pose.trans, dtype=np.float64), np.asarray(pose.root_trans, dtype=np.float64)[None]])
    return (torch.from_numpy(np.ascontiguousarray(q)).to(device), torch.from_numpy(np.ascontiguousarray(t)).to(device))


def lbs_deform(bundle, pose, device_avatars=None):
    """rig.py:107-146: deform the canonical cloud to a posed world-space cloud (on the GPU)."""
    j = int(np.asarray(bundle.lbs_weights).shape[1])
    if pose.n_joints != j:
        raise ContractViolation(f"pose has {pose.n_joints} joints, bundle has {j}")
    dav = device_avatars or DeviceAvatars([bundle])
    pq, pt = pose_tensors(pose, dav.device)
    pos, rot = skin_device(dav, 0, pq, pt)
    cloud = bundle.canonical
    return GaussianCloud(positions=pos.cpu().numpy(), sh_coeffs=cloud.sh_coeffs, opacities=cloud.opacities,
                         log_scales=cloud.log_scales, rotations=rot.cpu().numpy())


class AvatarRuntime:
    """An avatar instance inside a scene: bundle plus clocking/looping state (tasks.py:290-320)."""

    def __init__(self, bundle, start_offset=0.0, enabled=True, loop=True):
        self.bundle = bundle
        self.start_offset = float(start_offset)
        self.enabled = bool(enabled)
        self.loop = bool(loop)
        self._dev = None

    def clock(self, sim_time):
        t = self.start_offset + sim_time
        duration = self.bundle.duration
        if self.loop and duration > 0:
            return math.fmod(t, duration)
        return min(t, duration)

    def pose(self, sim_time):
        return sample_pose(self.bundle.trajectory, self.clock(sim_time))

    def root_xy_facing(self, sim_time):
        from .transforms import quat_to_matrix
        pose = self.pose(sim_time)
        xy = pose.root_trans[:2].copy()
        forward = quat_to_matrix(pose.root_quat) @ np.array([1.0, 0.0, 0.0])
        norm = np.linalg.norm(forward[:2])
        facing = forward[:2] / norm if norm > 1e-12 else np.array([1.0, 0.0])
        return xy, facing

    def deformed_cloud(self, sim_time):
        if self._dev is None:
            self._dev = DeviceAvatars([self.bundle])
        return lbs_deform(self.bundle, self.pose(sim_time), device_avatars=self._dev)
