"""the batched observation call of the episode loop (observe.BatchObserver,
tasks.py:498-504 + camera.agent_camera) and frame export from device frames (frame_io.py:11-58)."""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.camera import CameraDefaults, agent_camera, pose_world_to_camera


def test_agent_camera_matches_reference_formula():
    d = CameraDefaults(width=320, height=240, hfov_deg=90.0, near=0.1, far=100.0, mount_height=1.25)
    cam = agent_camera((1.5, -2.0), 0.7, d)
    np.testing.assert_array_equal(cam.world_to_camera, pose_world_to_camera(np.array([1.5, -2.0, 1.25]), 0.7))
    assert cam.fx == cam.fy == 160.0 / np.tan(np.radians(45.0)) and (cam.cx, cam.cy) == (160.0, 120.0)


@pytest.mark.gpu
def test_batch_observer_equals_per_episode_render_observation():
    from paper_2604_12626_b200.observe import BatchObserver
    box = S.room_box(1_000_000)
    scene = S.make_scene(80_000, box[0], box[1], seed=91)
    defaults = CameraDefaults(width=160, height=120, hfov_deg=90.0, near=0.1, far=100.0, mount_height=1.25)
    rng = np.random.default_rng(92)
    pos = rng.uniform(box[0][:2], box[1][:2], size=(4, 2))
    hd = rng.uniform(-np.pi, np.pi, size=4)
    obs = BatchObserver(scene, None, defaults, background=(0.1, 0.2, 0.3))
    out = obs.observe(pos, hd, quantized=True)
    for e in range(4):
        cam = agent_camera(pos[e], hd[e], defaults)
        o = O.render_observation(scene, [], cam, np.array([0.1, 0.2, 0.3]))
        assert np.abs(out["color"][e].cpu().numpy() - o.color).max() <= 2e-3
        hit = o.depth < cam.far
        d = out["depth"][e].cpu().numpy()
        assert (np.abs(d - o.depth) / o.depth)[hit].max(initial=0.0) <= 1e-4
    # the quantized payload follows frame_io's rule on the float frames, exactly
    c = out["color"].cpu().numpy().astype(np.float64)
    ref8 = (np.clip(c, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)
    np.testing.assert_array_equal(out["rgb8"].cpu().numpy(), ref8)
    np.testing.assert_array_equal(out["depth16"].cpu().numpy(), out["depth"].cpu().numpy().astype(np.float16))


@pytest.mark.gpu
def test_frame_export_formats(tmp_path):
    from PIL import Image
    from paper_2604_12626_b200 import frame_io as F
    rng = np.random.default_rng(93)
    color = rng.uniform(-0.2, 1.2, size=(37, 53, 3)).astype(np.float32)
    depth = rng.uniform(0.5, 9.0, size=(37, 53)).astype(np.float32)
    dc, dd = torch.from_numpy(color).cuda(), torch.from_numpy(depth).cuda()
    F.save_color_png(dc, tmp_path / "c.png")
    ref = (np.clip(color.astype(np.float64), 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)  # frame_io.py:13-14
    np.testing.assert_array_equal(np.asarray(Image.open(tmp_path / "c.png").convert("RGB")), ref)
    F.save_depth_pfm(dd, tmp_path / "d.pfm")
    raw = (tmp_path / "d.pfm").read_bytes()
    assert raw.startswith(b"Pf\n53 37\n-1.0\n")
    body = np.frombuffer(raw[len(b"Pf\n53 37\n-1.0\n"):], dtype="<f4").reshape(37, 53)
    np.testing.assert_array_equal(body, depth[::-1])  # bottom-to-top (frame_io.py:31)
    F.save_depth_f32(dd, tmp_path / "d.f32", 100.0)
    np.testing.assert_array_equal(np.fromfile(tmp_path / "d.f32", dtype="<f4").reshape(37, 53), depth)
