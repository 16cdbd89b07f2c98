"""A spatially ordered scene copy (DeviceCloud.spatially_ordered, sn_cloud ABI 3: rows in Morton
order, each row's original index, per-256-row block bounds) must render exactly like the original
order: the count kernel's whole-block depth decisions are only taken where every item would get the
same answer, and the order-dependent outputs -- depth ties (np.lexsort((idx, z)), renderer.py:80-101
via projection.py:184), gaussian ids -- use the original index."""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.camera import Camera
from paper_2604_12626_b200.cloud import GaussianCloud

pytestmark = pytest.mark.gpu

KEYS = ("color", "alpha", "depth", "contrib_scene", "stats")


def _tied_scene(n, planes, seed):
    """Gaussians on a few depth planes (world z) seen by axis-aligned cameras: camera z is exactly
    the world z plus a translation, so every plane is a run of exact depth ties whose reference order
    is the original index -- which the Morton order scrambles."""
    rng = np.random.default_rng(seed)
    base = S.make_scene(n, (-3.0, -2.0, 0.0), (3.0, 2.0, 1.0), seed=seed)
    pos = np.asarray(base.positions, dtype=np.float64).copy()
    pos[:, 2] = rng.choice(np.linspace(2.0, 6.0, planes), size=n)
    return GaussianCloud(pos.astype(np.float32), base.sh_coeffs, base.opacities, base.log_scales,
                         base.rotations).validate()


def _axis_cameras(k, w=320, h=240):
    cams = []
    for i in range(k):
        m = np.eye(4)
        m[:3, 3] = (0.3 * i - 0.5, 0.1 * i, -0.05 * i)
        cams.append(Camera.from_hfov(w, h, 70.0, 0.1, 20.0, m))
    return cams


def _render(cloud, cams, bg, **kw):
    from paper_2604_12626_b200 import _native as N
    from paper_2604_12626_b200 import renderer as R
    ctx = N.Context()
    out = None
    for _ in range(2):
        out = R.render_frames(cloud, cams, bg, contrib=True, context=ctx, **kw)
    torch.cuda.synchronize()
    return out, ctx


@pytest.mark.parametrize("views,stats,near_slice", [(True, True, 0), (False, True, 0), (False, False, 50),
                                                    (False, False, -1)])
def test_spatial_order_renders_like_original(views, stats, near_slice):
    from paper_2604_12626_b200.device import DeviceCloud
    scene = _tied_scene(600_000, 9, seed=311)
    cams = _axis_cameras(6)
    bg = np.array([0.2, 0.3, 0.4])
    orig = DeviceCloud(scene)
    sp = orig.spatially_ordered()
    assert sp.index is not None and not torch.equal(sp.index.cpu(), torch.arange(sp.n, dtype=torch.int32))
    a, ca = _render(orig, cams, bg, views=views, stats=stats, near_slice=near_slice)
    b, cb = _render(sp, cams, bg, views=views, stats=stats, near_slice=near_slice)
    for k in KEYS:
        if k in a:
            assert torch.equal(a[k], b[k]), k
    if views:  # the depth order's gaussian ids, per env
        from paper_2604_12626_b200 import renderer as R
        for e in (0, 5):
            ia = R.pass_intermediates(0, e, context=ca)["ids"]
            ib = R.pass_intermediates(0, e, context=cb)["ids"]
            np.testing.assert_array_equal(ia, ib)


def test_spatial_order_matches_oracle_with_ties():
    from paper_2604_12626_b200.device import DeviceCloud
    scene = _tied_scene(60_000, 5, seed=313)
    cams = _axis_cameras(2, 160, 120)
    bg = np.array([0.5, 0.5, 0.5])
    got, _ = _render(DeviceCloud(scene).spatially_ordered(), cams, bg, views=False, stats=True, near_slice=0)
    for e in range(2):
        o = O.rasterize(scene, cams[e], bg)
        np.testing.assert_array_equal(got["contrib_scene"][e].cpu().numpy(), o.contrib)
        assert got["stats"][e].tolist() == [o.stats[k] for k in ("n_input", "n_culled_depth", "n_culled_frame",
                                                                 "n_degenerate", "n_drawn")]
        assert np.abs(got["color"][e].cpu().numpy() - o.color).max() <= 2e-3


def test_spatial_copy_round_trips_to_host():
    from paper_2604_12626_b200.device import DeviceCloud
    scene = S.make_scene(5_000, (0, 0, 0), (4, 4, 2), seed=317)
    d = DeviceCloud(scene)
    s = d.spatially_ordered()
    for x, y in zip(d.to_host(), s.to_host()):
        np.testing.assert_array_equal(x, y)
    bb = s.block_bounds.cpu().numpy()
    pos = s.pos_opacity[:, :3].cpu().numpy()
    for blk in range(bb.shape[0]):
        p = pos[256 * blk: 256 * (blk + 1)]
        assert (p >= bb[blk, :3]).all() and (p <= bb[blk, 3:6]).all()
