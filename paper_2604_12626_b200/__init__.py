"""paper_2604_12626_b200 -- B200-native splat-observation hot path of Habitat-GS.

A drop-in for the reference package's renderer and avatar entry points
(/root/reference/pkg/src/splatnav: renderer.py, rig.py, raster/, tasks.AvatarRuntime): the same
signatures, backed by hand-written sm_100a CUDA kernels behind a C ABI
(include/splatnav_b200.h, libsplatnav_b200.so). Batched multi-environment rendering lives in
batch.BatchRenderer; multi-GPU env sharding in parallel.
"""

__version__ = "0.1.0"

from .avatar import AvatarBundle, Skeleton, Trajectory
from .camera import Camera, CameraDefaults, agent_camera, pose_world_to_camera
from .cloud import GaussianCloud, concat_clouds, empty_cloud
from .errors import ConsistencyError, ContractViolation, NativeError, SplatNavError, ValidationError

_LAZY = {
    "FrameRGBD": "renderer", "RenderStats": "renderer", "rasterize": "renderer", "rasterize_reference": "renderer",
    "composite": "renderer", "render_observation": "renderer",
    "JointPose": "rig", "sample_pose": "rig", "lbs_deform": "rig", "AvatarRuntime": "rig",
    "BatchRenderer": "batch", "DeviceCloud": "device", "DeviceAvatars": "device",
}


def __getattr__(name):
    # torch-backed modules load on first use so that containers/synthetic import without torch
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)
