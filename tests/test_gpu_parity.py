"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the reference's golden
fixtures on identical inputs.

Bars (BASELINE.json north_star):
* bit-exact: depth-sorted ids, tile CSR (tile_starts + per-tile depth ranks), per-pixel
  contributor counts, RenderStats;
* RGB max-abs error <= 2e-3; depth relative error <= 1e-4 (where alpha > 0; far elsewhere).
"""

import numpy as np
import pytest
import torch

from conftest import load_cases
from oracle import oracle as O
from paper_2604_12626_b200 import synthetic as S

pytestmark = pytest.mark.gpu

RGB_TOL = 2e-3
DEPTH_REL_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2604_12626_b200 import build
    build.build()


def R():
    from paper_2604_12626_b200 import renderer
    return renderer


def check_frame(color, alpha, depth, ref_color, ref_alpha, ref_depth, far):
    color = np.asarray(color, dtype=np.float64)
    depth = np.asarray(depth, dtype=np.float64)
    assert np.abs(color - ref_color).max() <= RGB_TOL, np.abs(color - ref_color).max()
    if ref_alpha is not None:
        assert np.abs(np.asarray(alpha, dtype=np.float64) - ref_alpha).max() <= RGB_TOL
    hit = ref_depth < far
    rel = np.abs(depth - ref_depth) / np.maximum(np.abs(ref_depth), 1e-12)
    assert rel[hit].max(initial=0.0) <= DEPTH_REL_TOL, rel[hit].max(initial=0.0)
    np.testing.assert_array_equal(depth[~hit], ref_depth[~hit].astype(np.float32).astype(np.float64))


def check_discrete(case_ids, tile_starts, pair_splat, contrib, pass_id, env, n_tiles, context=None):
    r = R()
    inter = r.pass_intermediates(pass_id, env, context=context)
    np.testing.assert_array_equal(inter["ids"], case_ids)
    if tile_starts is not None:
        ts, ps = r.tile_csr(n_tiles, pass_id, env, context=context)
        np.testing.assert_array_equal(ts, tile_starts)
        if pair_splat is not None:
            np.testing.assert_array_equal(ps, pair_splat)
    return inter


def render_case(case, cloud, cam):
    r = R()
    out = r.render_frames(cloud, [cam], case.background(), contrib=True)
    return {k: v.cpu().numpy() for k, v in out.items() if isinstance(v, torch.Tensor)}


def _check_golden_case(case, cloud, cam):
    out = render_case(case, cloud, cam)
    tiles_x, tiles_y = O.tiles_for(cam.width, cam.height)
    inter = check_discrete(case["ids"], case["tile_starts"], case.get("pair_splat"), None, 0, 0, tiles_x * tiles_y)
    np.testing.assert_array_equal(out["contrib_scene"][0], case["contrib"].astype(np.int32))
    assert out["stats"][0].tolist() == case["stats"].tolist()
    np.testing.assert_array_equal(inter["depths"], case["depths"])
    if "means2d" in case and case["ids"].size:
        np.testing.assert_array_equal(inter["means2d"], case["means2d"])
        assert np.abs(inter["colors"] - case["colors"]).max() <= 1e-5
    check_frame(out["color"][0], out["alpha"][0] if "alpha" in case else None, out["depth"][0], case["color"],
                case.get("alpha"), case["depth"], cam.far)


@pytest.mark.parametrize("name", ["c1_scenes", "edges"])
def test_golden_small(name):
    for case in load_cases(name):
        _check_golden_case(case, case.cloud(), case.camera())


def test_golden_config0():
    (case,) = load_cases("config0")
    scene, cam = S.config0()
    _check_golden_case(case, scene, cam)


def test_golden_room_batched():
    cases = load_cases("room")
    box = S.room_box(1_000_000)
    scene = S.make_scene(100_000, box[0], box[1], seed=5)
    cams = S.room_cameras(2, box, seed=6)
    out = R().render_frames(scene, cams, np.array([1.0, 1.0, 1.0]), contrib=True)
    tiles_x, tiles_y = O.tiles_for(640, 480)
    for e, case in enumerate(cases):
        check_discrete(case["ids"], case["tile_starts"], None, None, 0, e, tiles_x * tiles_y)
        np.testing.assert_array_equal(out["contrib_scene"][e].cpu().numpy(), case["contrib"].astype(np.int32))
        check_frame(out["color"][e].cpu().numpy(), None, out["depth"][e].cpu().numpy(), case["color"], None,
                    case["depth"].astype(np.float64), cams[e].far)


def _oracle_check_env(out, e, cloud, cam, bg, pass_id=0, layer_mode=False, context=None):
    o = O.rasterize(cloud, cam, None if layer_mode else bg)
    proj = O.project_cloud(cloud, cam)
    tiles_x, tiles_y = O.tiles_for(cam.width, cam.height)
    ts, ps = O.bin_tiles(proj.means2d, proj.radii, tiles_x, tiles_y)
    check_discrete(proj.ids.astype(np.int32), ts, ps, None, pass_id, e, tiles_x * tiles_y, context=context)
    key = "contrib_scene" if pass_id == 0 else "contrib_layer"
    np.testing.assert_array_equal(out[key][e].cpu().numpy(), o.contrib)
    return o


def test_batched_envs_match_oracle_near_001_and_01():
    box = S.room_box(1_000_000)
    scene = S.make_scene(150_000, box[0], box[1], seed=21)
    for near in (0.1, 0.01):
        cams = S.room_cameras(6, box, seed=22, near=near)
        bg = np.array([0.3, 0.6, 0.9])
        out = R().render_frames(scene, cams, bg, contrib=True)
        for e in (0, 3, 5):
            o = _oracle_check_env(out, e, scene, cams[e], bg)
            check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                        o.color, o.alpha, o.depth, cams[e].far)
            assert out["stats"][e].tolist() == [o.stats[k] for k in ("n_input", "n_culled_depth", "n_culled_frame",
                                                                     "n_degenerate", "n_drawn")]


def test_float64_cloud_and_layer_mode():
    box = S.room_box(1_000_000)
    scene = S.make_scene(30_000, box[0], box[1], seed=31)
    scene.positions = scene.positions.astype(np.float64) + 1e-9  # not float32-representable -> f64 path
    cams = S.room_cameras(2, box, seed=32, width=160, height=120)
    out = R().render_frames(scene, cams, None, contrib=True)
    for e in range(2):
        o = _oracle_check_env(out, e, scene, cams[e], None, layer_mode=True)
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o.color, o.alpha, o.depth, cams[e].far)


def test_rasterize_reference_equals_tiled():
    case = load_cases("c1_scenes")[3]
    r = R()
    cloud, cam, bg = case.cloud(), case.camera(), case.background()
    a = r.render_frames(cloud, [cam], bg, tiled=True, contrib=True)
    b = r.render_frames(cloud, [cam], bg, tiled=False, contrib=True)
    assert torch.equal(a["color"], b["color"]) and torch.equal(a["depth"], b["depth"])
    assert torch.equal(a["contrib_scene"], b["contrib_scene"])
    ref = r.rasterize_reference(cloud, cam, bg)
    assert np.abs(ref.color - case["color"]).max() <= RGB_TOL


def test_drop_in_rasterize_and_stats():
    from paper_2604_12626_b200.renderer import RenderStats
    case = load_cases("edges")[2]  # degenerate splats
    stats = RenderStats()
    frame = R().rasterize(case.cloud(), case.camera(), case.background(), stats=stats)
    assert [stats.n_input, stats.n_culled_depth, stats.n_culled_frame, stats.n_degenerate, stats.n_drawn] == \
        case["stats"].tolist()
    assert frame.color.dtype == np.float64 and frame.shape == (64, 64)
    assert np.abs(frame.color - case["color"]).max() <= RGB_TOL


def test_determinism_bit_identical():
    box = S.room_box(1_000_000)
    scene = S.make_scene(50_000, box[0], box[1], seed=41)
    cams = S.room_cameras(3, box, seed=42)
    r = R()
    a = r.render_frames(scene, cams, np.ones(3))
    b = r.render_frames(scene, cams, np.ones(3))
    for k in ("color", "alpha", "depth"):
        assert torch.equal(a[k], b[k])


# ------------------------------------------------------------------------------ avatars


def _avatar_setup(n_avatars=2, n_gauss=3000, seed=50):
    box = S.room_box(1_000_000)
    bundles = [S.make_avatar(n_gauss, seed=seed + i, n_frames=12, floor_lo=(1.0, 1.0), floor_hi=(7.0, 7.0))
               for i in range(n_avatars)]
    return box, bundles


def test_sample_pose_and_lbs_bit_exact_vs_oracle():
    from paper_2604_12626_b200 import rig
    _, bundles = _avatar_setup(1)
    b = bundles[0]
    for t in (0.0, 0.1, 0.137, 0.2, 99.0):
        pose = rig.sample_pose(b.trajectory, t)
        oq, ot = O.sample_pose(b.trajectory.quats, b.trajectory.trans, b.trajectory.fps, t)
        np.testing.assert_array_equal(np.concatenate([pose.quats, pose.root_quat[None]]), oq)
        np.testing.assert_array_equal(np.concatenate([pose.trans, pose.root_trans[None]]), ot)
        cloud = rig.lbs_deform(b, pose)
        op, orr = O.lbs_deform(b.canonical.positions, b.canonical.rotations, b.lbs_weights, b.inv_bind, oq, ot)
        assert np.abs(cloud.positions - op).max() <= 1e-12
        assert np.abs(cloud.rotations - orr).max() <= 1e-12


def test_lbs_golden_fixtures():
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.avatar import AvatarBundle, Skeleton, Trajectory
    from paper_2604_12626_b200.cloud import GaussianCloud
    for case in load_cases("lbs"):
        traj = Trajectory(float(case["fps"]), case["traj_quats"], case["traj_trans"])
        pose = rig.sample_pose(traj, float(case["t"]))
        np.testing.assert_array_equal(np.concatenate([pose.quats, pose.root_quat[None]]), case["pose_quats"])
        np.testing.assert_array_equal(np.concatenate([pose.trans, pose.root_trans[None]]), case["pose_trans"])
        n, j = case["weights"].shape
        canon = GaussianCloud(case["canon_positions"], np.zeros((n, 1, 3), np.float32), np.zeros(n, np.float32),
                              np.zeros((n, 3), np.float32), case["canon_rotations"])
        bundle = AvatarBundle(canon, case["weights"], case["inv_bind"],
                              Skeleton(np.array([-1] + [0] * (j - 1)), np.zeros((j, 3))), traj)
        out = rig.lbs_deform(bundle, pose)
        assert np.abs(out.positions - case["out_positions"]).max() <= 1e-12
        assert np.abs(out.rotations - case["out_rotations"]).max() <= 1e-12


def test_render_observation_golden():
    r = R()
    for case in load_cases("observation"):
        avatars = [case.cloud(f"avatar{i}_") for i in range(int(case["n_avatars"]))]
        frame = r.render_observation(case.cloud("scene_"), avatars, case.camera(), case["background"])
        check_frame(frame.color, frame.alpha, frame.depth, case["color"], case["alpha"], case["depth"],
                    case.camera().far)


@pytest.mark.parametrize("exact", [False, True])
def test_fused_avatar_batch_matches_oracle(exact):
    """Batched scene + 2 skinned avatars at per-env times vs the oracle fed the GPU-skinned clouds,
    through the float32 chain with bounds (exact=False) and through the float64 walk for every
    pixel (exact=True)."""
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.batch import BatchRenderer
    from paper_2604_12626_b200.cloud import concat_clouds
    box, bundles = _avatar_setup(2, 4000)
    scene = S.make_scene(60_000, box[0], box[1], seed=61)
    cams = S.room_cameras(5, box, seed=62, width=320, height=240)
    # point two cameras at the avatars so the layer is non-trivial
    times = np.array([0.0, 0.05, 0.133, 0.21, 0.3])
    br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.1], loops=[1, 0], background=(0.2, 0.3, 0.4))
    out = br.render(cams, times, contrib=True, stats=True, exact=exact)
    for e in range(len(cams)):
        clouds = []
        for a, b in enumerate(bundles):
            rt = rig.AvatarRuntime(b, start_offset=[0.0, 0.1][a], loop=[True, False][a])
            clouds.append(rt.deformed_cloud(float(times[e])))
        layer = concat_clouds(clouds)
        o = O.render_observation(scene, clouds, cams[e], np.array([0.2, 0.3, 0.4]))
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o.color, o.alpha, o.depth, cams[e].far)
        # discrete parity of the avatar layer pass
        lo = O.rasterize(layer, cams[e], None)
        np.testing.assert_array_equal(out["contrib_layer"][e].cpu().numpy(), lo.contrib)
        proj = O.project_cloud(layer, cams[e])
        inter = R().pass_intermediates(1, e, context=br.context)
        np.testing.assert_array_equal(inter["ids"], proj.ids.astype(np.int32))


def test_composite_kernel_exact():
    rng = np.random.default_rng(3)
    h, w = 17, 23

    def frame():
        return R().FrameRGBD(rng.uniform(size=(h, w, 3)), rng.uniform(size=(h, w)), rng.uniform(0.5, 5, size=(h, w)))

    f, b = frame(), frame()
    f.alpha[0, :5] = 0.5
    got = R().composite(f, b)
    ref = O.composite(f, b)
    np.testing.assert_array_equal(got.color, ref.color)
    np.testing.assert_array_equal(got.depth, ref.depth)
    np.testing.assert_array_equal(got.alpha, ref.alpha)


def test_blend_tile_range_plugin():
    from paper_2604_12626_b200 import raster
    case = load_cases("c1_scenes")[5]
    k = raster.get_kernel("cuda")
    assert k.KERNEL_NAME == "cuda"
    with pytest.raises(ValueError):
        raster.get_kernel("python")
    proj = O.project_cloud(case.cloud(), case.camera())
    ts, ps = O.bin_tiles(proj.means2d, proj.radii, 4, 4)
    acc = [np.zeros((64, 64, 3)), np.zeros((64, 64)), np.ones((64, 64)), np.zeros((64, 64))]
    k.blend_tile_range(0, 16, 4, 16, 64, 64, ts, ps, proj.means2d, proj.conics, proj.depths, proj.colors,
                       proj.alphas, *acc)
    ref = O.blend(4, 16, 64, 64, ts, ps, proj.means2d, proj.conics, proj.depths, proj.colors, proj.alphas)
    for a, b in zip(acc, ref[:4]):
        assert np.abs(a - b).max() <= 1e-12


def test_streaming_and_list_binners_agree():
    """Rect streaming (no lists) and materialized radix lists: the tile lists the blend actually
    consumes (sn_get_device_tiles -- the streamed per-tile queues vs the radix-sorted pairs) and the
    frames are identical."""
    box = S.room_box(1_000_000)
    scene = S.make_scene(120_000, box[0], box[1], seed=71)
    cams = S.room_cameras(5, box, seed=72, near=0.01)
    r = R()
    a = r.render_frames(scene, cams, np.ones(3), contrib=True, binning=0)
    csr_a = [r.device_tiles(1200, 0, e) for e in range(5)]
    b = r.render_frames(scene, cams, np.ones(3), contrib=True, binning=1)
    csr_b = [r.device_tiles(1200, 0, e) for e in range(5)]
    for (ta, pa), (tb, pb) in zip(csr_a, csr_b):
        np.testing.assert_array_equal(ta, tb)
        np.testing.assert_array_equal(pa, pb)
    for k in ("color", "alpha", "depth", "contrib_scene"):
        assert torch.equal(a[k], b[k])


def test_layer_pass_both_binners_agree():
    from paper_2604_12626_b200.batch import BatchRenderer
    box, bundles = _avatar_setup(2, 3000)
    scene = S.make_scene(40_000, box[0], box[1], seed=81)
    cams = S.room_cameras(4, box, seed=82, width=320, height=240)
    times = np.array([0.0, 0.07, 0.11, 0.3])
    br = BatchRenderer(scene, bundles, background=(0.5, 0.5, 0.5))
    outs = [R().render_frames(br.scene, cams, br.background, avatars=br.avatars, sim_times=times,
                              context=br.context, contrib=True, binning=m) for m in (0, 1, -1)]
    for o in outs[1:]:
        for k in ("color", "alpha", "depth", "contrib_scene", "contrib_layer"):
            assert torch.equal(outs[0][k], o[k]), k


def test_env_chunking_beyond_64_envs():
    """E > 64 runs in env chunks (key space); every env must still match the oracle exactly."""
    box = S.room_box(1_000_000)
    scene = S.make_scene(25_000, box[0], box[1], seed=91)
    cams = S.room_cameras(70, box, seed=92, width=48, height=40)
    bg = np.array([0.1, 0.2, 0.3])
    out = R().render_frames(scene, cams, bg, contrib=True)
    for e in range(70):
        o = O.rasterize(scene, cams[e], bg)
        np.testing.assert_array_equal(out["contrib_scene"][e].cpu().numpy(), o.contrib)
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o.color, o.alpha, o.depth, cams[e].far)


def test_avatar_active_mask_and_clock():
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.batch import BatchRenderer
    box, bundles = _avatar_setup(3, 2500, seed=95)
    scene = S.make_scene(30_000, box[0], box[1], seed=96)
    cams = S.room_cameras(4, box, seed=97, width=160, height=120)
    times = np.array([0.05, 0.5, 1.7, 3.3])  # past the 12-frame trajectories: loop vs clamp
    offs, loops = [0.0, 0.25, 0.6], [1, 0, 1]
    active = torch.tensor([[1, 1, 1], [0, 1, 0], [1, 0, 1], [0, 0, 0]], dtype=torch.uint8)
    br = BatchRenderer(scene, bundles, start_offsets=offs, loops=loops, background=(0.5, 0.4, 0.3))
    out = br.render(cams, times, avatar_active=active, contrib=True)
    for e in range(4):
        clouds = [rig.AvatarRuntime(b, start_offset=offs[a], loop=bool(loops[a])).deformed_cloud(float(times[e]))
                  for a, b in enumerate(bundles) if active[e, a]]
        o = O.render_observation(scene, clouds, cams[e], np.array([0.5, 0.4, 0.3]))
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o.color, o.alpha, o.depth, cams[e].far)


def test_negative_sample_time_is_a_contract_violation():
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.batch import BatchRenderer
    from paper_2604_12626_b200.errors import ContractViolation
    box, bundles = _avatar_setup(1, 500, seed=98)
    br = BatchRenderer(S.make_scene(1000, box[0], box[1], seed=1), bundles, loops=[0])
    cams = S.room_cameras(1, box, seed=2, width=32, height=32)
    with pytest.raises(ContractViolation):
        br.render(cams, np.array([-0.5]))
    with pytest.raises(ContractViolation):
        rig.sample_pose(bundles[0].trajectory, -0.1)


def test_full_size_config2_spot_check():
    """BASELINE config 2 at full size (1M scene, 4 x 50k avatars, 64 envs, 640x480): two envs
    against the oracle, discrete outputs exact."""
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.batch import BatchRenderer
    cfg = S.baseline_config(2, seed=0)
    offs = [0.37 * i for i in range(4)]
    br = BatchRenderer(cfg["scene"], cfg["avatars"], start_offsets=offs, background=(1.0, 1.0, 1.0))
    times = np.random.default_rng(5).uniform(0.0, 2.0, size=64)
    out = br.render(cfg["cameras"], times, contrib=True, stats=True)
    for e in (0, 41):
        cam = cfg["cameras"][e]
        clouds = [rig.AvatarRuntime(b, start_offset=offs[a]).deformed_cloud(float(times[e]))
                  for a, b in enumerate(cfg["avatars"])]
        o = O.render_observation(cfg["scene"], clouds, cam, np.ones(3))
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o.color, o.alpha, o.depth, cam.far)
        np.testing.assert_array_equal(out["contrib_scene"][e].cpu().numpy(), o.scene.contrib)
        np.testing.assert_array_equal(out["contrib_layer"][e].cpu().numpy(), o.layer.contrib)
        proj = O.project_cloud(cfg["scene"], cam)
        inter = R().pass_intermediates(0, e, context=br.context)
        np.testing.assert_array_equal(inter["ids"], proj.ids.astype(np.int32))


def test_3m_scene_spot_check():
    """BASELINE config 3/4 scale (3M gaussians in a 3x-area room): one env exact vs the oracle."""
    box = S.room_box(3_000_000)
    scene = S.make_scene(3_000_000, box[0], box[1], seed=7)
    cams = S.room_cameras(8, box, seed=8)
    out = R().render_frames(scene, cams, np.ones(3), contrib=True)
    o = O.rasterize(scene, cams[5], np.ones(3))
    np.testing.assert_array_equal(out["contrib_scene"][5].cpu().numpy(), o.contrib)
    check_frame(out["color"][5].cpu().numpy(), out["alpha"][5].cpu().numpy(), out["depth"][5].cpu().numpy(),
                o.color, o.alpha, o.depth, cams[5].far)


def test_fast_exp_error_budget():
    """The float32 blend chain's error budget (csrc/sn_blend.cu kEpsExp = 5e-7) assumes the fast
    exponential's relative error, argument rounding included, is <= 3.5e-7 over d2 in [0, 9.5]
    (measured: 2.76e-7); check it on the device."""
    from paper_2604_12626_b200 import _native as N
    err = N.selftest_fast_exp()
    assert 0.0 < err <= 3.5e-7, err


def test_exact_mode_agrees_with_fast_path():
    """The float32 chain's discrete outputs equal the all-float64 walk's, pixel for pixel; the
    continuous ones differ by float32 rounding only."""
    box = S.room_box(1_000_000)
    scene = S.make_scene(200_000, box[0], box[1], seed=71)
    cams = S.room_cameras(4, box, seed=72)
    bg = np.array([1.0, 1.0, 1.0])
    from paper_2604_12626_b200 import _native as N
    ctx_fast, ctx_exact = N.Context(), N.Context()
    fast = R().render_frames(scene, cams, bg, contrib=True, context=ctx_fast)
    ex = R().render_frames(scene, cams, bg, contrib=True, context=ctx_exact, exact=True)
    assert torch.equal(fast["contrib_scene"], ex["contrib_scene"])
    assert float((fast["color"] - ex["color"]).abs().max()) <= 1e-5
    rel = ((fast["depth"] - ex["depth"]).abs() / ex["depth"]).max()
    assert float(rel) <= 1e-5
    o = _oracle_check_env(ex, 1, scene, cams[1], bg, context=ctx_exact)
    check_frame(ex["color"][1].cpu().numpy(), ex["alpha"][1].cpu().numpy(), ex["depth"][1].cpu().numpy(),
                o.color, o.alpha, o.depth, cams[1].far)


def test_capacity_growth_rerenders_exactly():
    """A context sized by a small render must grow (one re-run) for a larger one and still give the
    oracle's discrete outputs."""
    from paper_2604_12626_b200 import _native as N
    box = S.room_box(1_000_000)
    small = S.make_scene(5_000, box[0], box[1], seed=81)
    big = S.make_scene(120_000, box[0], box[1], seed=82)
    cams = S.room_cameras(2, box, seed=83, width=320, height=240)
    bg = np.array([0.5, 0.5, 0.5])
    ctx = N.Context()
    R().render_frames(small, cams, bg, context=ctx)
    r0 = ctx.render_retries()
    out = R().render_frames(big, cams, bg, contrib=True, context=ctx)
    assert ctx.render_retries() > r0
    for e in range(2):
        o = _oracle_check_env(out, e, big, cams[e], bg, context=ctx)
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o.color, o.alpha, o.depth, cams[e].far)


def test_env_chunking_with_avatar_layer():
    """E > 64 with the avatar layer: chunks are rendered scene then layer (the layer's fixups read the
    same chunk's scene workspace); every env's observation must match the oracle fed the GPU-skinned
    clouds, and the layer's contributor counts must be exact."""
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.batch import BatchRenderer
    from paper_2604_12626_b200.cloud import concat_clouds
    box, bundles = _avatar_setup(2, 2500, seed=71)
    scene = S.make_scene(20_000, box[0], box[1], seed=72)
    cams = S.room_cameras(70, box, seed=73, width=48, height=40)
    times = np.linspace(0.0, 0.35, 70)
    br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.05], loops=[1, 1], background=(0.3, 0.3, 0.3))
    out = br.render(cams, times, contrib=True, stats=True)
    keys = ("n_input", "n_culled_depth", "n_culled_frame", "n_degenerate", "n_drawn")
    for e in (0, 31, 63, 64, 69):
        clouds = [rig.AvatarRuntime(b, start_offset=[0.0, 0.05][a], loop=True).deformed_cloud(float(times[e]))
                  for a, b in enumerate(bundles)]
        o = O.render_observation(scene, clouds, cams[e], np.array([0.3, 0.3, 0.3]))
        check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                    o.color, o.alpha, o.depth, cams[e].far)
        lo = O.rasterize(concat_clouds(clouds), cams[e], None)
        np.testing.assert_array_equal(out["contrib_layer"][e].cpu().numpy(), lo.contrib)
        # RenderStats over both passes (the whole-avatar culls are counted in their categories)
        so = O.rasterize(scene, cams[e], np.array([0.3, 0.3, 0.3]))
        assert out["stats"][e].tolist() == [so.stats[k] + lo.stats[k] for k in keys]


def test_degenerate_and_extreme_splats():
    """Huge, needle-thin and non-finite-scale splats (the float32 chain's worst conditioning and the
    degenerate path) against the oracle, fast path and exact mode."""
    from paper_2604_12626_b200 import _native as N
    box = S.room_box(1_000_000)
    scene = S.make_scene(40_000, box[0], box[1], seed=81)
    rng = np.random.default_rng(82)
    ls = scene.log_scales.copy()
    ls[:300] = np.stack([rng.uniform(-1.0, 0.5, 300), rng.uniform(-9.0, -7.0, 300), rng.uniform(-9, -7, 300)], 1)
    ls[300:310] = 400.0  # overflow -> non-finite covariance -> degenerate (projection.py:44-51,154)
    scene.log_scales = ls.astype(np.float32)
    cams = S.room_cameras(3, box, seed=83, width=160, height=120, near=0.01)
    bg = np.array([1.0, 1.0, 1.0])
    for exact in (False, True):
        ctx = N.Context()
        out = R().render_frames(scene, cams, bg, contrib=True, context=ctx, exact=exact)
        for e in range(3):
            o = _oracle_check_env(out, e, scene, cams[e], bg, context=ctx)
            check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                        o.color, o.alpha, o.depth, cams[e].far)
            assert out["stats"][e].tolist() == [o.stats[k] for k in ("n_input", "n_culled_depth", "n_culled_frame",
                                                                     "n_degenerate", "n_drawn")]


def test_async_render_pipeline_matches_sync_and_retries():
    """sn_render_async / sn_render_wait: renders queued back to back (the next one before the host
    waits for the previous) give frames bit-identical to synchronous renders; on a fresh context the
    first check asks for a retry (workspace growth) and the re-queued render matches; a
    third render while two are in flight is refused."""
    from paper_2604_12626_b200 import _native as N
    from paper_2604_12626_b200.batch import BatchRenderer, HostPipeline
    box, bundles = _avatar_setup(2, 2500, seed=91)
    scene = S.make_scene(30_000, box[0], box[1], seed=92)
    bg = (0.4, 0.4, 0.4)
    sets = [(S.room_cameras(3, box, seed=93 + s, width=64, height=48), np.linspace(0.05 * s, 0.3, 3)) for s in range(4)]
    ref = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.1], loops=[1, 1], background=bg)
    want = []
    for cams, times in sets:
        o = ref.render(cams, times)
        want.append({k: o[k].clone() for k in ("color", "alpha", "depth")})
    br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.1], loops=[1, 1], background=bg, context=N.Context())
    outs = [{k: torch.empty_like(v) for k, v in w.items()} for w in want]
    br.render(*sets[0], out=outs[0], wait=False)
    assert br.context.render_wait()  # empty workspace: this render overflowed and must be re-queued
    for cams, times in sets:  # grow the workspace to fit every set (synchronous renders retry inside)
        br.render(cams, times)
    br.render(*sets[0], out=outs[0], wait=False)
    assert not br.context.render_wait()
    br.render(*sets[1], out=outs[1], wait=False)
    br.render(*sets[2], out=outs[2], wait=False)
    from paper_2604_12626_b200.errors import ContractViolation
    with pytest.raises(ContractViolation):
        br.render(*sets[3], out=outs[3], wait=False)
    assert not br.context.render_wait()
    br.render(*sets[3], out=outs[3], wait=False)
    assert not br.context.render_wait()
    assert not br.context.render_wait()
    for got, exp in zip(outs, want):
        for k in exp:
            assert torch.equal(got[k], exp[k]), k
    # the host pipeline (async renders, downloads overlapped) delivers the same frames -- on a warm
    # context, and on a fresh one whose first checks ask for retries (its re-render path)
    fresh = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.1], loops=[1, 1], background=bg, context=N.Context())
    for renderer in (br, fresh):
        pipe = HostPipeline(renderer, 3, 48, 64)
        r0 = renderer.context.render_retries()
        for st in sets:
            pipe.submit(*st)
        pipe.wait()
        for i in (len(sets) - 2, len(sets) - 1):
            for k in want[i]:
                assert torch.equal(pipe.host[i % 2][k], want[i][k].cpu()), (k, i)
        if renderer is fresh:
            assert renderer.context.render_retries() > r0


@pytest.mark.parametrize("seed", [101, 202, 303])
def test_random_scale_spread_against_oracle(seed):
    """Seeded scenes with a wide spread of scales and opacities (tiny to frame-filling splats, needle
    and disc shapes) and small frames, near 0.1 and 0.01: the tight rectangles, the warp-block
    separating axes and the float32 chain must leave every discrete output equal to the oracle's."""
    box = S.room_box(1_000_000)
    scene = S.make_scene(20_000, box[0], box[1], seed=seed)
    rng = np.random.default_rng(seed + 1)
    scene.log_scales = rng.normal(-3.0, 1.5, scene.log_scales.shape).astype(np.float32)
    scene.opacities = rng.normal(0.5, 2.0, scene.opacities.shape).astype(np.float32)
    for near in (0.1, 0.01):
        cams = S.room_cameras(3, box, seed=seed + 2, width=96, height=80, near=near)
        bg = np.array([0.2, 0.5, 0.8])
        out = R().render_frames(scene, cams, bg, contrib=True)
        for e in range(3):
            o = _oracle_check_env(out, e, scene, cams[e], bg)
            check_frame(out["color"][e].cpu().numpy(), out["alpha"][e].cpu().numpy(), out["depth"][e].cpu().numpy(),
                        o.color, o.alpha, o.depth, cams[e].far)
            assert out["stats"][e].tolist() == [o.stats[k] for k in ("n_input", "n_culled_depth", "n_culled_frame",
                                                                     "n_degenerate", "n_drawn")]


def test_whole_avatar_visibility_code():
    """An avatar whose bounding ball projects strictly inside the frame and depth range is kept
    without per-gaussian skinning in the count (code kWholeVisible = 4): the layer's kept set,
    order and contributor counts must still be the oracle's."""
    import ctypes
    from paper_2604_12626_b200 import _native as N
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.batch import BatchRenderer
    from paper_2604_12626_b200.camera import Camera, pose_world_to_camera
    from paper_2604_12626_b200.cloud import concat_clouds
    box = S.room_box(1_000_000)
    scene = S.make_scene(30_000, box[0], box[1], seed=301)
    bundles = [S.make_avatar(3000, seed=302, n_frames=6, floor_lo=(4.0, 4.0), floor_hi=(4.0, 4.0))]
    cams = [Camera.from_hfov(320, 240, 90.0, 0.1, 100.0, pose_world_to_camera(np.array([x, 4.0, 1.25]), 0.0))
            for x in (0.5, 1.0, 0.0)]
    times = np.array([0.0, 0.05, 0.1])
    br = BatchRenderer(scene, bundles, background=(0.5, 0.5, 0.5))
    out = br.render(cams, times, contrib=True, stats=True)
    codes = (ctypes.c_uint8 * 3)()
    lib = ctypes.CDLL(N.LIB_PATH)
    assert lib.sn_debug_avatar_codes(br.context.handle, codes, ctypes.c_int64(3)) == 0
    assert 4 in list(codes), list(codes)  # the whole-visible path was taken
    for e in range(3):
        clouds = [rig.AvatarRuntime(bundles[0]).deformed_cloud(float(times[e]))]
        layer = concat_clouds(clouds)
        lo = O.rasterize(layer, cams[e], None)
        np.testing.assert_array_equal(out["contrib_layer"][e].cpu().numpy(), lo.contrib)
        proj = O.project_cloud(layer, cams[e])
        inter = R().pass_intermediates(1, e, context=br.context)
        np.testing.assert_array_equal(inter["ids"], proj.ids.astype(np.int32))
