"""Batched entry point: E independent environments per call (the throughput path).

BatchRenderer keeps the scene and the avatar set resident on one GPU and renders a batch of
cameras (one per env) with per-env avatar sim times in one sn_render call: scene pass, fused
skin->project avatar-layer pass, compositor in the blend epilogue. Outputs stay on the device as
torch tensors (E,H,W,3) / (E,H,W) / (E,H,W).
"""

import os

import numpy as np
import torch

from . import _native as N
from .device import DeviceAvatars, DeviceCloud
from .renderer import render_frames


class BatchRenderer:
    def __init__(self, scene, avatars=None, start_offsets=None, loops=None, background=(1.0, 1.0, 1.0), device=None,
                 context=None, spatial=None):
        """spatial: keep the scene as a spatially ordered copy (DeviceCloud.spatially_ordered; the same
        frames, ids and stats as the original order, fewer per-(gaussian, env) depth tests); default
        on (SPLATNAV_SPATIAL=0 turns the default off)."""
        if spatial is None:
            spatial = os.environ.get("SPLATNAV_SPATIAL", "1") != "0"
        self.scene = DeviceCloud.wrap(scene, device)
        if spatial:
            self.scene = self.scene.spatially_ordered()
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

    def render(self, cameras, sim_times=None, avatar_active=None, tiled=True, contrib=False, stats=False,
               exact=False, out=None, wait=True, payload=False, serialize=False, stage_ms=None, work=None,
               binning=-1, views=True, near_slice=-1):
        """wait=False: queue the render and return (see render_frames); pair every such call with
        a later self.context.render_wait(). payload=True also returns the uint8 / fp16 observation
        payload (rgb8, depth16) written by the render's epilogues."""
        if self.avatars is not None and sim_times is None:
            sim_times = np.zeros(len(cameras))
        return render_frames(self.scene, cameras, self.background, avatars=self.avatars, sim_times=sim_times,
                             tiled=tiled, context=self.context, contrib=contrib, stats=stats,
                             avatar_active=avatar_active, exact=exact, out=out, wait=wait, payload=payload,
                             serialize=serialize, stage_ms=stage_ms, work=work, binning=binning, views=views,
                             near_slice=near_slice)

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


class HostPipeline:
    """Render batches straight into pinned host memory with the device->host copies of batch i
    overlapped with the render of batch i+1 (double-buffered, separate copy stream). Renders are
    queued with sn_render_async and checked one submit later, so the host never idles the GPU
    between batches; a render whose check asks for a retry (workspace growth) is re-rendered
    synchronously, with any render queued after it.

    submit(cameras, sim_times) -> slot index; the frames of a slot are valid in host[slot] after
    wait(slot), until the slot is reused two submits later."""

    FRAME_KEYS = ("color", "alpha", "depth")
    PAYLOAD_KEYS = ("rgb8", "depth16")

    def __init__(self, renderer, n_envs, height, width, depth=2, payload=False):
        """payload=True downloads the uint8 RGB + fp16 depth observation payload the render writes
        (frame_io's rule) instead of the float32 frames."""
        self.r = renderer
        self.payload = payload
        self.KEYS = self.PAYLOAD_KEYS if payload else self.FRAME_KEYS
        dev = renderer.device
        # renders on their own stream, not the legacy default stream (whose implicit
        # synchronization would serialize them with the copies)
        self.render_stream = torch.cuda.Stream(dev)
        self.copy_stream = torch.cuda.Stream(dev)
        shapes = {"color": ((n_envs, height, width, 3), torch.float32), "alpha": ((n_envs, height, width), torch.float32),
                  "depth": ((n_envs, height, width), torch.float32),
                  "rgb8": ((n_envs, height, width, 3), torch.uint8), "depth16": ((n_envs, height, width), torch.float16)}
        self.host = [{k: torch.empty(shapes[k][0], dtype=shapes[k][1], pin_memory=True) for k in self.KEYS}
                     for _ in range(depth)]
        # device frames of each slot, rendered into in place: no allocation per step (a caching-
        # allocator miss would cudaMalloc / cudaFree and serialize the render with the copies)
        dkeys = self.FRAME_KEYS + (self.PAYLOAD_KEYS if payload else ())
        self.dev = [{k: torch.empty(shapes[k][0], dtype=shapes[k][1], device=dev) for k in dkeys}
                    for _ in range(depth)]
        self.bytes_per_submit = sum(t.numel() * t.element_size() for t in self.host[0].values())
        self.done = [None] * depth
        self.pending = []  # (slot, cameras, sim_times, ready event) queued, not yet checked
        self.i = 0

    def submit(self, cameras, sim_times=None):
        slot = self.i % len(self.host)
        self.i += 1
        with torch.cuda.stream(self.render_stream):
            if self.done[slot] is not None:
                # the render overwrites this slot's device frames once their download (two submits
                # back) is done: a device-side wait, so the host keeps queueing ahead of the GPU
                self.render_stream.wait_event(self.done[slot])
            out = self.r.render(cameras, sim_times, out=dict(self.dev[slot]), wait=False, payload=self.payload,
                                views=False)
            ready = torch.cuda.Event()
            ready.record(self.render_stream)
        self.dev[slot] = {k: out[k] for k in self.dev[slot]}  # the tensors the render writes
        self.pending.append((slot, cameras, sim_times, ready))
        if len(self.pending) > 1:
            self._retire()
        return slot

    def _copy(self, slot, ready):
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(ready)
            for k in self.KEYS:
                self.host[slot][k].copy_(self.dev[slot][k], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self.done[slot] = ev

    def _retire(self):
        """Check the oldest queued render and start its download."""
        slot, cams, times, ready = self.pending.pop(0)
        if not self.r.context.render_wait():
            self._copy(slot, ready)
            return
        # the workspace grew: this render and those queued after it ran on the old capacities
        redo = [(slot, cams, times)] + [(s, c, t) for s, c, t, _ in self.pending]
        for _ in self.pending:
            self.r.context.render_wait()
        self.pending = []
        for s, c, t in redo:
            with torch.cuda.stream(self.render_stream):
                out = self.r.render(c, t, out=dict(self.dev[s]), payload=self.payload, views=False)
                self.dev[s] = {k: out[k] for k in self.dev[s]}
                ev = torch.cuda.Event()
                ev.record(self.render_stream)
            self._copy(s, ev)

    def wait(self, slot=None):
        while self.pending:
            self._retire()
        for i, ev in enumerate(self.done):
            if ev is not None and (slot is None or i == slot):
                ev.synchronize()
                torch.cuda.current_stream(self.r.device).wait_event(ev)
        return self.host[slot] if slot is not None else None


def quantize_observation(color, depth):
    """uint8 RGB (x*255+0.5, frame_io.py:13-14) + fp16 depth, the gather payload (one CUDA kernel,
    sn_quantize_frames)."""
    from .frame_io import quantize
    return quantize(color, depth)
