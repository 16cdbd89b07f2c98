"""Parity at the configurations and code paths the round-1 tests did not reach:
* BASELINE config 3 at full size: a 6M-gaussian scene, 256 envs at 640x480 (four 64-env chunks),
  envs in the first, a middle and the last chunk against the oracle: depth-sorted ids, contributor
  counts, RenderStats, frames;
* BASELINE config 4's shape: 1,024 envs x 16 skinned 50k-gaussian avatars (small frames), envs 0,
  511 and 1,023: layer contributor counts and depth order exact, RenderStats over both passes;
* avatars smaller than a CTA (60-200 gaussians), so one 256-gaussian block spans >= 3 avatars and
  the skinning reads the poses it could not stage from global memory;
* transmittance stacks built so the reference's sequential float64 T lands within a few ulps of
  the 1e-4 cutoff (_kernels_cy.pyx:65-66,86), on both sides: the contributor counts of the float32
  chain (with its float64 fixups) and of the all-float64 mode must equal the oracle's.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2604_12626_b200 import synthetic as S

pytestmark = pytest.mark.gpu

RGB_TOL = 2e-3
DEPTH_REL_TOL = 1e-4
KEYS = ("n_input", "n_culled_depth", "n_culled_frame", "n_degenerate", "n_drawn")


def check_frame(color, alpha, depth, o, far):
    color = np.asarray(color, dtype=np.float64)
    depth = np.asarray(depth, dtype=np.float64)
    assert np.abs(color - o.color).max() <= RGB_TOL
    assert np.abs(np.asarray(alpha, dtype=np.float64) - o.alpha).max() <= RGB_TOL
    hit = o.depth < far
    rel = np.abs(depth - o.depth) / np.maximum(np.abs(o.depth), 1e-12)
    assert rel[hit].max(initial=0.0) <= DEPTH_REL_TOL


def test_config3_6m_256_envs():
    from paper_2604_12626_b200 import _native as N
    from paper_2604_12626_b200 import renderer as R
    n = 6_000_000
    box = S.room_box(n)
    scene = S.make_scene(n, box[0], box[1], seed=3)
    cams = S.room_cameras(256, box, seed=4)
    bg = np.ones(3)
    ctx = N.Context()
    out = R.render_frames(scene, cams, bg, contrib=True, stats=True, context=ctx)
    torch.cuda.synchronize()
    for e in (5, 130, 255):  # first, third and last 64-env chunk (255: the views cover the last chunk)
        o = O.rasterize(scene, cams[e], bg)
        np.testing.assert_array_equal(out["contrib_scene"][e].cpu().numpy(), o.contrib)
        assert out["stats"][e].tolist() == [o.stats[k] for k in KEYS]
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o, cams[e].far)
        if e == 255:
            proj = O.project_cloud(scene, cams[e])
            np.testing.assert_array_equal(R.pass_intermediates(0, e, context=ctx)["ids"], proj.ids.astype(np.int32))
    # the throughput path at this scale: depth-sliced (auto), with RenderStats and without them (the
    # lazy far classification) -- bit-identical to the unsliced render above, every env
    for stats in (True, False):
        for _ in range(2):  # (the first may grow the far capacities)
            sl = R.render_frames(scene, cams, bg, contrib=True, stats=stats, views=False, context=ctx)
        torch.cuda.synchronize()
        for k in ("color", "alpha", "depth", "contrib_scene") + (("stats",) if stats else ()):
            assert torch.equal(sl[k], out[k]), (stats, k)


def _layer_checks(out, br, bundles, offs, scene, cams, times, envs, bg):
    from paper_2604_12626_b200 import renderer as R
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.cloud import concat_clouds
    for e in envs:
        clouds = [rig.AvatarRuntime(b, start_offset=offs[a]).deformed_cloud(float(times[e]))
                  for a, b in enumerate(bundles)]
        o = O.render_observation(scene, clouds, cams[e], bg)
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o, cams[e].far)
        layer = concat_clouds(clouds)
        lo = O.rasterize(layer, cams[e], None)
        np.testing.assert_array_equal(out["contrib_layer"][e].cpu().numpy(), lo.contrib)
        so = O.rasterize(scene, cams[e], bg)
        np.testing.assert_array_equal(out["contrib_scene"][e].cpu().numpy(), so.contrib)
        assert out["stats"][e].tolist() == [so.stats[k] + lo.stats[k] for k in KEYS]
        if e == envs[-1]:  # the harness views hold the last env chunk
            proj = O.project_cloud(layer, cams[e])
            np.testing.assert_array_equal(R.pass_intermediates(1, e, context=br.context)["ids"],
                                          proj.ids.astype(np.int32))


def test_config4_shape_1024_envs_16_avatars():
    from paper_2604_12626_b200.batch import BatchRenderer
    box = S.room_box(1_000_000)
    scene = S.make_scene(200_000, box[0], box[1], seed=41)
    bundles = [S.make_avatar(50_000, seed=420 + i, n_frames=16, floor_lo=box[0][:2], floor_hi=box[1][:2])
               for i in range(16)]
    cams = S.room_cameras(1024, box, seed=43, width=96, height=72)
    times = np.random.default_rng(44).uniform(0.0, 1.0, size=1024)
    offs = [0.05 * i for i in range(16)]
    bg = np.array([0.7, 0.7, 0.7])
    br = BatchRenderer(scene, bundles, start_offsets=offs, background=bg)
    out = br.render(cams, times, contrib=True, stats=True)
    _layer_checks(out, br, bundles, offs, scene, cams, times, (0, 511, 1023), bg)
    assert int(out["contrib_layer"].sum()) > 0  # the layer is not empty across the batch
    # the throughput path over all 1,024 envs: lean views and a forced 5% depth slice, with and
    # without RenderStats -- the same decisions (contributor counts, stats), colours within float32
    # rounding of the composite's float64 recomputes (see tests/test_slicing.py)
    for stats in (True, False):
        for _ in range(2):
            sl = br.render(cams, times, contrib=True, stats=stats, views=False, near_slice=50)
        torch.cuda.synchronize()
        for k in ("contrib_scene", "contrib_layer") + (("stats",) if stats else ()):
            assert torch.equal(sl[k], out[k]), (stats, k)
        for k in ("color", "alpha"):
            assert (sl[k] - out[k]).abs().max().item() <= 2e-6, (stats, k)
        assert ((sl["depth"] - out["depth"]).abs() <= 5e-6 * out["depth"].abs()).all()


def test_avatars_smaller_than_a_block():
    """Eight avatars of 60-200 gaussians: a 256-gaussian CTA spans >= 3 of them, so the count
    kernel's pose staging (two avatars per block) misses some and skins them from global memory."""
    from paper_2604_12626_b200.batch import BatchRenderer
    box = S.room_box(1_000_000)
    sizes = [60, 200, 90, 75, 150, 64, 120, 99]
    assert any(sum(1 for a in range(8) if s0 < sum(sizes[:a + 1]) and sum(sizes[:a]) < s0 + 256) >= 3
               for s0 in range(0, sum(sizes), 256))
    bundles = [S.make_avatar(n, seed=500 + i, n_frames=10, floor_lo=(3.0, 3.0), floor_hi=(5.0, 5.0))
               for i, n in enumerate(sizes)]
    for b in bundles:  # larger splats so these small clouds cover pixels
        b.canonical.log_scales = (b.canonical.log_scales + 1.5).astype(np.float32)
    scene = S.make_scene(10_000, box[0], box[1], seed=51)
    from paper_2604_12626_b200.camera import Camera, pose_world_to_camera
    cams = [Camera.from_hfov(128, 96, 90.0, 0.1, 100.0, pose_world_to_camera(np.array([x, y, 1.0]), yaw))
            for x, y, yaw in ((1.5, 1.5, 0.78), (6.5, 6.5, -2.36), (1.5, 6.5, -0.78), (4.0, 0.5, 1.57),
                              (0.5, 4.0, 0.0))]
    times = np.linspace(0.0, 0.3, len(cams))
    offs = [0.03 * i for i in range(8)]
    bg = np.array([0.2, 0.2, 0.2])
    br = BatchRenderer(scene, bundles, start_offsets=offs, background=bg)
    for exact in (False, True):
        out = br.render(cams, times, contrib=True, stats=True, exact=exact)
        _layer_checks(out, br, bundles, offs, scene, cams, times, tuple(range(len(cams))), bg)
    assert int(out["contrib_layer"].sum()) > 1000


# ------------------------------------------------------------------ near-cutoff transmittance stacks

def _libm_exp():
    import ctypes
    import ctypes.util
    lib = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
    lib.exp.restype = ctypes.c_double
    lib.exp.argtypes = [ctypes.c_double]
    return lib.exp


def _cutoff_stacks(seed=7, grid=28, spacing=9, window=8):
    """Stacks of splats centred exactly on a pixel centre (d2 = 0, so exp(-d2/2) = 1 in any
    implementation): base splats with random alphas leave T_prev in [1.05e-4, 1.5e-4], then a
    critical splat with a small alpha whose float64 opacity is logit(1 - 1e-4 / T_prev) moved by
    -window..window ulps (one stack per offset, same base), then 3 splats behind it (the first counted only
    while T >= 1e-4). One ulp of the critical opacity moves T by ~0.3 ulp of 1e-4, so the stacks of
    each base straddle the cutoff within a few ulps whatever exp (numpy's, glibc's or the device's,
    which differ by an ulp on a few percent of arguments) turns the opacities into alphas.
    Camera: f = 128 px, centre (128, 128), looking down -z from the origin; a point (x, y, -1)
    projects exactly to (128 x + 128, -128 y + 128). Returns the cloud, the camera and the stack
    pixels (stack order = index order)."""
    from paper_2604_12626_b200.camera import Camera
    from paper_2604_12626_b200.cloud import GaussianCloud
    rng = np.random.default_rng(seed)
    pos, opa, pix = [], [], []
    k = 0
    base = None
    for gy in range(grid):
        for gx in range(grid):
            px, py = 6 + gx * spacing, 6 + gy * spacing
            x, y = (px + 0.5 - 128.0) / 128.0, -(py + 0.5 - 128.0) / 128.0
            j = k % (2 * window + 1)
            if j == 0:
                # base alphas until T drops below 1.5e-4 (12-60 splats: some stacks cross a
                # 32-contribution group of the fixup walk), the last one set so T_prev lands in
                # [1.05e-4, 1.5e-4]
                a = rng.uniform(0.05, rng.choice([0.3, 0.6]), size=200)
                t = np.cumprod(1.0 - a)
                L = int(np.searchsorted(-t, -1.5e-4)) + 1
                target = rng.uniform(1.05e-4, 1.5e-4)
                a[L - 1] = 1.0 - target / (t[L - 2] if L > 1 else 1.0)
                ac = 1.0 - 1e-4 / target
                base = (list(np.log(a[:L] / (1.0 - a[:L]))), float(np.log(ac / (1.0 - ac))))
            o_base, o0 = base
            oc = o0 + (j - window) * float(np.spacing(abs(o0)))
            for o in list(o_base) + [oc, 0.3, -0.2, 0.8]:
                pos.append((x, y, -1.0))
                opa.append(float(o))
            pix.append((py, px))
            k += 1
    n = len(pos)
    cloud = GaussianCloud(np.array(pos, dtype=np.float64), np.full((n, 1, 3), 0.1, dtype=np.float64),
                          np.array(opa, dtype=np.float64), np.full((n, 3), -12.0), np.tile([1.0, 0, 0, 0], (n, 1)))
    w2c = np.diag([1.0, -1.0, -1.0, 1.0])
    cam = Camera(128.0, 128.0, 128.0, 128.0, 256, 256, 0.01, 100.0, w2c)
    return cloud, cam, pix


def _critical_t(proj, pix):
    """Per stack, the sequential float64 T after its critical splat (_kernels_cy.pyx:86), from the
    given projection's alphas (all splats share z, so depth order = index order)."""
    order = np.argsort(proj.ids, kind="stable")
    alphas, means = proj.alphas[order], proj.means2d[order]
    crit, i = [], 0
    for (py, px) in pix:
        j = i
        while j < means.shape[0] and means[j, 0] == px + 0.5 and means[j, 1] == py + 0.5:
            j += 1
        T = 1.0
        for a in alphas[i:j - 3]:
            T = T * (1.0 - min(a, 0.99))
        crit.append(T)
        i = j
    assert i == means.shape[0]
    return np.array(crit)


def test_transmittance_cutoff_within_ulps():
    """The float32 chain must hand these pixels to the float64 fixup, whose walk must take the
    reference's sequential decision. Checked against the oracle's blend (pinned bit-for-bit to the
    reference's compiled kernel) run on the device's own projected splats, and against the oracle's
    full render where the two projections agree."""
    from paper_2604_12626_b200 import _native as N
    from paper_2604_12626_b200 import renderer as R
    cloud, cam, pix = _cutoff_stacks()
    ulp = np.spacing(1e-4)
    bg = np.array([1.0, 1.0, 1.0])
    o = O.rasterize(cloud, cam, bg)
    for exact in (False, True):
        ctx = N.Context()
        out = R.render_frames(cloud, [cam], bg, contrib=True, context=ctx, exact=exact)
        got = out["contrib_scene"][0].cpu().numpy()
        inter = R.pass_intermediates(0, 0, context=ctx)
        class P:
            pass
        dp = P()
        dp.ids, dp.alphas, dp.means2d = inter["ids"], inter["alphas"], inter["means2d"]
        crit = _critical_t(dp, pix)
        near_below = ((crit < 1e-4) & (crit >= 1e-4 - 2 * ulp)).sum()
        near_above = ((crit >= 1e-4) & (crit <= 1e-4 + 2 * ulp)).sum()
        assert near_below >= 100 and near_above >= 100, (near_below, near_above)
        ts, ps = R.tile_csr(256, 0, 0, context=ctx)
        ref = O.blend(16, 16, 256, 256, ts, ps, inter["means2d"], inter["conics"], inter["depths"], inter["colors"],
                      inter["alphas"])
        np.testing.assert_array_equal(got, ref[4])  # the reference blend's sequential decisions
        # base splats + the critical one, + the first splat behind it while T >= 1e-4 (which then stops)
        want = np.array([len(s) for s in _stack_sizes(inter, pix)]) - 3 + (crit >= 1e-4)
        np.testing.assert_array_equal(np.array([got[py, px] for py, px in pix]), want)
        # against the oracle's own projection where both computed the same alphas for a stack
        same = _same_alpha_stacks(inter, O.project_cloud(cloud, cam), pix)
        assert same.sum() >= 200
        for s_i in np.nonzero(same)[0]:
            py, px = pix[s_i]
            assert got[py, px] == o.contrib[py, px]
        check_frame(out["color"][0].cpu().numpy(), out["alpha"][0].cpu().numpy(), out["depth"][0].cpu().numpy(),
                    o, cam.far)


def _stack_sizes(inter, pix):
    order = np.argsort(inter["ids"], kind="stable")
    means = inter["means2d"][order]
    out, i = [], 0
    for (py, px) in pix:
        j = i
        while j < means.shape[0] and means[j, 0] == px + 0.5 and means[j, 1] == py + 0.5:
            j += 1
        out.append(range(i, j))
        i = j
    return out


def _same_alpha_stacks(inter, proj, pix):
    a = inter["alphas"][np.argsort(inter["ids"], kind="stable")]
    b = proj.alphas[np.argsort(proj.ids, kind="stable")]
    return np.array([np.array_equal(a[list(r)], b[list(r)]) for r in _stack_sizes(inter, pix)])
