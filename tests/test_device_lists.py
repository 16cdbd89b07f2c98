"""The tile lists the device blend actually consumes (sn_get_device_tiles), against the oracle's
_bin_tiles (renderer.py:80-101). The device keeps, per tile, only the splats whose TIGHT rectangle
(the support ellipse's bounding box) covers it. So every device list must be:
* an in-order sub-list of the reference list (same depth ranks, same order), and
* a superset of the splats that have an in-frame pixel of the tile inside their support
  (d2 <= 9 with the reference's float64 d2, _kernels_cy.pyx:73-75) -- the only ones the blend can
  accumulate.
Both the streamed lists of the scene pass and the radix binner's (env, tile) lists (the avatar
layer, or binning=1) are checked, over multi-env chunks."""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2604_12626_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _needed(proj, ts, ps, tiles_x, width, height):
    """Per pair of the reference CSR: does the splat reach an in-frame pixel of the tile (d2 <= 9)?"""
    need = np.zeros(ps.shape[0], dtype=bool)
    m, c = proj.means2d, proj.conics
    for t in range(ts.shape[0] - 1):
        a, b = int(ts[t]), int(ts[t + 1])
        if a == b:
            continue
        x0, y0 = (t % tiles_x) * 16, (t // tiles_x) * 16
        xs = np.arange(x0, min(x0 + 16, width)) + 0.5
        ys = np.arange(y0, min(y0 + 16, height)) + 0.5
        px, py = np.meshgrid(xs, ys)
        px, py = px.ravel()[None, :], py.ravel()[None, :]
        sid = ps[a:b]
        dx = m[sid, 0][:, None] - px
        dy = m[sid, 1][:, None] - py
        ca, cb, cc = c[sid, 0][:, None], c[sid, 1][:, None], c[sid, 2][:, None]
        d2 = ca * dx * dx + 2.0 * cb * dx * dy + cc * dy * dy
        need[a:b] = (~(d2 > 9.0)).any(axis=1)
    return need


def check_env_lists(dev_ts, dev_ranks, cloud, cam, label):
    proj = O.project_cloud(cloud, cam)
    tiles_x, tiles_y = O.tiles_for(cam.width, cam.height)
    ts, ps = O.bin_tiles(proj.means2d, proj.radii, tiles_x, tiles_y)
    need = _needed(proj, ts, ps, tiles_x, cam.width, cam.height)
    assert dev_ts.shape == ts.shape
    kept_total = 0
    for t in range(ts.shape[0] - 1):
        ref = ps[ts[t]:ts[t + 1]]
        got = dev_ranks[dev_ts[t]:dev_ts[t + 1]]
        # in-order sub-list of the reference list
        pos = np.searchsorted(ref, got)  # reference lists are ascending in depth rank
        assert np.all(np.diff(got) > 0), (label, t)
        assert np.all(pos < ref.size) and np.array_equal(ref[np.minimum(pos, ref.size - 1)], got), (label, t)
        # every splat with a pixel of the tile inside its support is kept
        missing = np.setdiff1d(ref[need[ts[t]:ts[t + 1]]], got)
        assert missing.size == 0, (label, t, missing[:5])
        kept_total += got.size
    return kept_total, ps.size


def test_scene_streamed_and_radix_lists_match_oracle():
    from paper_2604_12626_b200 import _native as N
    from paper_2604_12626_b200 import renderer as R
    scene, cam = S.config0()
    box = S.room_box(1_000_000)
    room = S.make_scene(120_000, box[0], box[1], seed=131)
    for near in (0.01, 0.1):
        cams = S.room_cameras(5, box, seed=132, width=160, height=120, near=near)
        lists = {}
        for binning in (0, 1):
            ctx = N.Context()
            R.render_frames(room, cams, np.ones(3), binning=binning, context=ctx)
            lists[binning] = [R.device_tiles(80, 0, e, context=ctx) for e in range(5)]
        for e in (0, 2, 4):
            # both binners hand the blend the same tight lists
            np.testing.assert_array_equal(lists[0][e][0], lists[1][e][0])
            np.testing.assert_array_equal(lists[0][e][1], lists[1][e][1])
            kept, total = check_env_lists(*lists[0][e], room, cams[e], f"room near={near} env {e}")
            assert 0 < kept <= total
    ctx = N.Context()
    R.render_frames(scene, [cam], np.zeros(3), context=ctx)
    kept, total = check_env_lists(*R.device_tiles(256, 0, 0, context=ctx), scene, cam, "config0")
    assert kept < total  # the tight rectangles drop reference pairs that reach no pixel


def test_layer_radix_lists_match_oracle():
    """The avatar layer's (env | tile) radix-sorted lists over a 4-env chunk, vs _bin_tiles of the
    GPU-skinned layer cloud."""
    from paper_2604_12626_b200 import renderer as R
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.batch import BatchRenderer
    from paper_2604_12626_b200.cloud import concat_clouds
    box = S.room_box(1_000_000)
    bundles = [S.make_avatar(3000, seed=141 + i, n_frames=12, floor_lo=(3.0, 3.0), floor_hi=(5.0, 5.0))
               for i in range(3)]
    scene = S.make_scene(20_000, box[0], box[1], seed=144)
    cams = []
    for i, (x, y, yaw) in enumerate([(1.0, 1.0, 0.8), (7.0, 7.0, -2.3), (1.0, 7.0, -0.8), (4.0, 1.0, 1.57)]):
        from paper_2604_12626_b200.camera import Camera, pose_world_to_camera
        cams.append(Camera.from_hfov(160, 120, 90.0, 0.1, 100.0, pose_world_to_camera(np.array([x, y, 1.25]), yaw)))
    times = np.array([0.0, 0.1, 0.2, 0.3])
    br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.1, 0.2], background=(0.5, 0.5, 0.5))
    br.render(cams, times)
    nonempty = 0
    for e in range(4):
        clouds = [rig.AvatarRuntime(b, start_offset=0.1 * a).deformed_cloud(float(times[e]))
                  for a, b in enumerate(bundles)]
        layer = concat_clouds(clouds)
        ts, ranks = R.device_tiles(80, 1, e, context=br.context)
        kept, total = check_env_lists(ts, ranks, layer, cams[e], f"layer env {e}")
        nonempty += kept > 0
    assert nonempty >= 2
