"""The observation consumer of the episode loop, batched.

tasks.step_episode renders one observation per call (tasks.py:498-504):

    camera = agent_camera(agent.position, agent.heading, scene.camera_defaults)   # camera.py:80-90
    avatar_clouds = [a.deformed_cloud(state.sim_time) for a in avatars]          # tasks.py:319
    rgbd = render_observation(scene.cloud, avatar_clouds, camera, scene.background)

BatchObserver does exactly that for E episodes in one sn_render call: the agent cameras are built
host-side (a few hundred bytes), the avatars are skinned on the device at each episode's sim time
with AvatarRuntime's clock (start offset, loop), and the frames stay on the device -- optionally
quantized there to the uint8 RGB + fp16 depth observation payload.
"""

import numpy as np

from .batch import BatchRenderer
from .camera import CameraDefaults, agent_camera
from .frame_io import quantize


class BatchObserver:
    def __init__(self, scene_cloud, avatars=None, camera_defaults=None, background=(1.0, 1.0, 1.0),
                 start_offsets=None, loops=None, device=None, context=None):
        self.defaults = camera_defaults or CameraDefaults()
        self.renderer = BatchRenderer(scene_cloud, avatars, start_offsets=start_offsets, loops=loops,
                                      background=background, device=device, context=context)

    def cameras(self, positions, headings):
        pos = np.asarray(positions, dtype=np.float64).reshape(-1, 2)
        hd = np.asarray(headings, dtype=np.float64).reshape(-1)
        if pos.shape[0] != hd.shape[0]:
            raise ValueError(f"{pos.shape[0]} positions but {hd.shape[0]} headings")
        return [agent_camera(pos[e], float(hd[e]), self.defaults) for e in range(hd.shape[0])]

    def observe(self, positions, headings, sim_times=None, quantized=False, contrib=False):
        """Observations of E agents at (x, y) positions and headings (radians), avatars at per-episode
        sim times. Returns device tensors: color (E,H,W,3), alpha, depth (float32) and, when
        `quantized`, rgb8 (E,H,W,3) uint8 and depth16 (E,H,W) float16."""
        cams = self.cameras(positions, headings)
        times = None if sim_times is None else np.asarray(sim_times, dtype=np.float64).reshape(-1)
        out = self.renderer.render(cams, times, contrib=contrib)
        if quantized:
            out["rgb8"], out["depth16"] = quantize(out["color"], out["depth"])
        return out
