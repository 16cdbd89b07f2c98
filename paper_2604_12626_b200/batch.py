"""Batched entry point: E independent environments per call (the throughput path).

BatchRenderer keeps the scene and the avatar set resident on one GPU and renders a batch of
cameras (one per env) with per-env avatar sim times in one sn_render call: scene pass, fused
skin->project avatar-layer pass, compositor in the blend epilogue. Outputs stay on the device as
torch tensors (E,H,W,3) / (E,H,W) / (E,H,W).
"""

import numpy as np
import torch

from . import _native as N
from .device import DeviceAvatars, DeviceCloud
from .renderer import render_frames


class BatchRenderer:
    def __init__(self, scene, avatars=None, start_offsets=None, loops=None, background=(1.0, 1.0, 1.0), device=None,
                 context=None):
        self.scene = DeviceCloud.wrap(scene, device)
        if avatars is None or isinstance(avatars, DeviceAvatars):
            self.avatars = avatars
        else:
            avatars = list(avatars)
            self.avatars = DeviceAvatars(avatars, start_offsets, loops, device=self.scene.device) if avatars else None
        self.background = None if background is None else np.asarray(background, dtype=np.float64)
        self.context = context or N.Context()

    @property
    def device(self):
        return self.scene.device

    def render(self, cameras, sim_times=None, avatar_active=None, tiled=True, contrib=False, stats=False):
        if self.avatars is not None and sim_times is None:
            sim_times = np.zeros(len(cameras))
        return render_frames(self.scene, cameras, self.background, avatars=self.avatars, sim_times=sim_times,
                             tiled=tiled, context=self.context, contrib=contrib, stats=stats,
                             avatar_active=avatar_active)

    def render_to_host(self, cameras, sim_times=None, host_out=None):
        """render() followed by a device->host copy into pinned buffers (the end-to-end path)."""
        out = self.render(cameras, sim_times)
        if host_out is None:
            host_out = {k: torch.empty(out[k].shape, dtype=out[k].dtype, pin_memory=True)
                        for k in ("color", "alpha", "depth")}
        for k in ("color", "alpha", "depth"):
            host_out[k].copy_(out[k], non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return host_out


def quantize_observation(color, depth):
    """uint8 RGB (x*255+0.5, frame_io.py:13-14) + fp16 depth, the gather payload."""
    rgb = (color.clamp(0.0, 1.0) * 255.0 + 0.5).to(torch.uint8)
    return rgb, depth.to(torch.float16)
