"""Skins of any width (SURVEY.md 8(a) lbs_deform, rig.py:107-146) and the avatar-bundle validation
the reference performs (avatar.py:86-178): dense softmax weights over 24 / 55 joints take the CSR
influence layout; the reference-written fixtures are tests/golden/lbs_dense.npz and
tests/golden/assets/{bundle_dense55,bad_*} (tests/golden/make_dense.py)."""

import os

import numpy as np
import pytest
import torch

from conftest import REPO, load_cases
from oracle import oracle as O
from paper_2604_12626_b200 import assets as A
from paper_2604_12626_b200.avatar import AvatarBundle, CapsuleTrack, Skeleton, Trajectory
from paper_2604_12626_b200.cloud import GaussianCloud
from paper_2604_12626_b200.device import csr_influences, influence_widths
from paper_2604_12626_b200.errors import ValidationError

D = os.path.join(REPO, "tests", "golden", "assets")
E = np.load(os.path.join(D, "expected_dense.npz"))
LBS_TOL = 1e-12
BAD = ("bad_traj_nan", "bad_inv_bind_inf", "bad_capsule_nan", "bad_capsule_radius")


def _bundle(case):
    n, j = case["weights"].shape
    canon = GaussianCloud(case["canon_positions"], np.zeros((n, 1, 3), np.float32), np.zeros(n, np.float32),
                          np.zeros((n, 3), np.float32), case["canon_rotations"])
    traj = Trajectory(float(case["fps"]), case["traj_quats"], case["traj_trans"])
    return AvatarBundle(canon, case["weights"], case["inv_bind"], Skeleton(case["parents"], case["rest"]), traj)


# ------------------------------------------------------------------------------------- CPU

def test_csr_influences_roundtrip():
    rng = np.random.default_rng(3)
    dense = rng.uniform(size=(50, 55)) * (rng.uniform(size=(50, 55)) < 0.4)
    dense[7] = 0.0  # an all-zero row
    off, jj, ww = csr_influences(dense, row_offset=5)
    assert off[0] == 5 and off.dtype == np.uint32 and jj.dtype == np.uint8
    np.testing.assert_array_equal(np.diff(off.astype(np.int64)), influence_widths(dense))
    back = np.zeros_like(dense)
    for i in range(50):
        a, b = int(off[i]) - 5, int(off[i + 1]) - 5
        assert list(jj[a:b]) == sorted(jj[a:b])  # ascending joint order
        back[i, jj[a:b]] = ww[a:b]
    np.testing.assert_array_equal(back, dense)


def test_oracle_lbs_matches_reference_dense_skins():
    """The C oracle (dense, sequential FMA chains) against the reference's lbs_deform on dense 24 and
    55-joint skins: numpy/OpenBLAS sums some of these products in 8 interleaved accumulators at this
    row count, so agreement is to a few ulps (the 1e-12 LBS tolerance), not bit-for-bit."""
    for case in load_cases("lbs_dense"):
        q, t = O.sample_pose(case["traj_quats"], case["traj_trans"], float(case["fps"]), float(case["t"]))
        p, r = O.lbs_deform(case["canon_positions"], case["canon_rotations"], case["weights"], case["inv_bind"], q, t)
        assert np.abs(p - case["out_positions"]).max() <= LBS_TOL
        assert np.abs(r - case["out_rotations"]).max() <= LBS_TOL


@pytest.mark.parametrize("name", BAD)
def test_bad_bundles_host_checks_raise_reference_messages(name):
    """Trajectory / inverse-bind / capsule checks run on the host (the canonical cloud and weights
    are checked on the device first, like AvatarBundle.validate's order)."""
    s = A.read_bundle_dir(os.path.join(D, name))
    with pytest.raises(ValidationError) as ei:
        A._validate_host_parts(s)
        A._validate_capsules(s)
    assert f"ValidationError: {ei.value}" == str(E[f"{name}_message"])


def test_avatar_containers_validate_like_reference():
    case = load_cases("lbs_dense")[0]
    b = _bundle(case)
    b.validate()
    q = b.trajectory.quats.copy()
    q[2, 3, 1] = np.nan
    with pytest.raises(ValidationError, match="non-finite trajectory data"):
        Trajectory(b.trajectory.fps, q, b.trajectory.trans).validate()
    b2 = _bundle(case)
    b2.inv_bind = b2.inv_bind.copy()
    b2.inv_bind[1, 0, 3] = np.inf
    with pytest.raises(ValidationError, match="non-finite inverse bind matrices"):
        b2.validate()
    frames = np.ones((b.trajectory.n_frames, 2, 7))
    b3 = _bundle(case)
    b3.capsule_track = CapsuleTrack(frames.copy())
    b3.validate()
    frames[0, 1, 6] = 0.0
    b3.capsule_track = CapsuleTrack(frames)
    with pytest.raises(ValidationError, match="capsule radii must be positive"):
        b3.validate()


# ------------------------------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_lbs_dense_golden_fixtures():
    """lbs_deform through the CSR influence path on the device vs the reference's outputs."""
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200.device import DeviceAvatars
    for case in load_cases("lbs_dense"):
        b = _bundle(case)
        dav = DeviceAvatars([b])
        assert dav.infl is not None  # rows wider than 4: CSR layout
        pose = rig.sample_pose(b.trajectory, float(case["t"]))
        out = rig.lbs_deform(b, pose, device_avatars=dav)
        assert np.abs(out.positions - case["out_positions"]).max() <= LBS_TOL
        assert np.abs(out.rotations - case["out_rotations"]).max() <= LBS_TOL
        # and against the oracle at the same pose (both dense sequential chains)
        q = np.concatenate([pose.quats, pose.root_quat[None]])
        t = np.concatenate([pose.trans, pose.root_trans[None]])
        p, r = O.lbs_deform(b.canonical.positions, b.canonical.rotations, b.lbs_weights, b.inv_bind, q, t)
        assert np.abs(out.positions - p).max() <= LBS_TOL and np.abs(out.rotations - r).max() <= LBS_TOL


@pytest.mark.gpu
def test_dense_bundle_loads_like_reference():
    from paper_2604_12626_b200.device import DeviceAvatars
    dav = A.load_avatar_bundles([os.path.join(D, "bundle_dense55")])
    assert dav.n_joints == 55 and dav.infl is not None
    off, jj, ww = csr_influences(E["dense55_weights"])  # renormalized by the reference's loader
    n = dav.n
    np.testing.assert_array_equal(dav.infl[0].cpu().numpy().view(np.uint32), off)
    np.testing.assert_array_equal(dav.infl[1].cpu().numpy()[:off[-1]], jj)
    np.testing.assert_array_equal(dav.infl[2].cpu().numpy()[:off[-1]], ww)
    np.testing.assert_array_equal(dav.pos_opacity.cpu().numpy()[:n, :3], E["dense55_positions"].astype(np.float64))

    class B:
        pass
    b = B()
    b.canonical = GaussianCloud(E["dense55_positions"], E["dense55_sh_coeffs"], E["dense55_opacities"],
                                E["dense55_log_scales"], E["dense55_rotations"])
    b.lbs_weights, b.inv_bind = E["dense55_weights"], E["dense55_inv_bind"]
    b.trajectory = Trajectory(float(E["dense55_fps"]), E["dense55_traj_quats"], E["dense55_traj_trans"])
    host = DeviceAvatars([b])
    for i in range(3):
        assert torch.equal(dav.infl[i], host.infl[i]), i


@pytest.mark.gpu
@pytest.mark.parametrize("name", BAD)
def test_bad_bundles_raise_reference_messages(name):
    with pytest.raises(ValidationError) as ei:
        A.load_avatar_bundles([os.path.join(D, name)])
    assert f"ValidationError: {ei.value}" == str(E[f"{name}_message"])


@pytest.mark.gpu
@pytest.mark.parametrize("joints", [24, 55])
def test_fused_render_with_dense_skins_matches_oracle(joints):
    """The fused skin -> project avatar layer over CSR influences: frames vs the oracle fed the
    GPU-skinned clouds, layer contributor counts and depth order exact."""
    from paper_2604_12626_b200 import rig
    from paper_2604_12626_b200 import renderer as R
    from paper_2604_12626_b200 import synthetic as S
    from paper_2604_12626_b200.batch import BatchRenderer
    from paper_2604_12626_b200.cloud import concat_clouds
    box = S.room_box(1_000_000)
    bundles = [S.make_dense_avatar(1500, joints, seed=40 + i, floor_lo=(2.0, 2.0), floor_hi=(6.0, 6.0))
               for i in range(2)]
    scene = S.make_scene(20_000, box[0], box[1], seed=43)
    cams = S.room_cameras(3, box, seed=44, width=160, height=120)
    times = np.array([0.0, 0.21, 0.4])
    br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.1], background=(0.3, 0.3, 0.3))
    assert br.avatars.infl is not None
    out = br.render(cams, times, contrib=True, stats=True)
    for e in range(3):
        clouds = [rig.AvatarRuntime(b, start_offset=[0.0, 0.1][a]).deformed_cloud(float(times[e]))
                  for a, b in enumerate(bundles)]
        o = O.render_observation(scene, clouds, cams[e], np.array([0.3, 0.3, 0.3]))
        assert np.abs(out["color"][e].cpu().numpy() - o.color).max() <= 2e-3
        layer = concat_clouds(clouds)
        lo = O.rasterize(layer, cams[e], None)
        np.testing.assert_array_equal(out["contrib_layer"][e].cpu().numpy(), lo.contrib)
        proj = O.project_cloud(layer, cams[e])
        inter = R.pass_intermediates(1, e, context=br.context)
        np.testing.assert_array_equal(inter["ids"], proj.ids.astype(np.int32))
