"""Fixtures for skins wider than 4 influences and for the avatar-bundle validation errors, written
by the REFERENCE package (/root/reference/pkg/src/splatnav), in the build container only:

    python tests/golden/make_dense.py

* lbs_dense.npz: rig.sample_pose + rig.lbs_deform (rig.py:78-146) of avatars whose weight rows are
  dense softmax skins over 24 (SMPL) and 55 (SMPL-X-sized) joints -- every row has J nonzeros.
* assets/bundle_dense55/: a dense 55-joint bundle saved with avatar.save_avatar_bundle and the
  arrays avatar.load_avatar_bundle returns for it (expected_dense.npz), with rows off by 4e-5 so
  the float64 renormalization runs.
* assets/bad_*/: bundles the reference rejects (non-finite trajectory, non-finite inverse binds,
  non-finite capsules, non-positive capsule radius) and its exception text for each.
The avatars come from paper_2604_12626_b200.synthetic.make_dense_avatar (seeded); the reference
classes are rebuilt from its arrays.
"""
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from splatnav import avatar as RA  # noqa: E402
from splatnav import rig as RR  # noqa: E402
from splatnav.cloud import GaussianCloud as RCloud  # noqa: E402

from paper_2604_12626_b200 import synthetic as S  # noqa: E402

OUT = os.path.join(HERE, "assets")


def to_ref(b, capsules=None):
    c = b.canonical
    cloud = RCloud(c.positions, c.sh_coeffs, c.opacities, c.log_scales, c.rotations)
    skel = RA.Skeleton(np.asarray(b.skeleton.parents), np.asarray(b.skeleton.rest_positions))
    traj = RA.Trajectory(b.trajectory.fps, np.asarray(b.trajectory.quats), np.asarray(b.trajectory.trans))
    return RA.AvatarBundle(cloud, np.asarray(b.lbs_weights), np.asarray(b.inv_bind), skel, traj, capsules)


def gen_lbs():
    cases = []
    for j, n, seed in ((24, 600, 1), (55, 400, 2)):
        b = to_ref(S.make_dense_avatar(n, j, seed=seed, floor_lo=(1.0, 1.0), floor_hi=(3.0, 3.0))).validate()
        for t in (0.0, 0.117, 0.3):
            pose = RR.sample_pose(b.trajectory, t)
            cloud = RR.lbs_deform(b, pose)
            cases.append({
                "canon_positions": np.asarray(b.canonical.positions),
                "canon_rotations": np.asarray(b.canonical.rotations),
                "weights": np.asarray(b.lbs_weights), "inv_bind": np.asarray(b.inv_bind),
                "parents": np.asarray(b.skeleton.parents), "rest": np.asarray(b.skeleton.rest_positions),
                "traj_quats": b.trajectory.quats, "traj_trans": b.trajectory.trans,
                "fps": np.array(b.trajectory.fps), "t": np.array(t),
                "out_positions": cloud.positions, "out_rotations": cloud.rotations,
            })
    flat = {f"{i}/{k}": v for i, c in enumerate(cases) for k, v in c.items()}
    flat["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "lbs_dense.npz"), **flat)


def gen_bundles():
    expected = {}
    src = S.make_dense_avatar(300, 55, seed=7, sh_degree=2, floor_lo=(1.0, 1.0), floor_hi=(3.0, 3.0))
    b = to_ref(src, RR.bake_capsules(RA.Skeleton(np.asarray(src.skeleton.parents),
                                                 np.asarray(src.skeleton.rest_positions)),
                                     RA.Trajectory(src.trajectory.fps, np.asarray(src.trajectory.quats),
                                                   np.asarray(src.trajectory.trans))))
    b.lbs_weights = b.lbs_weights * 1.00004
    d = os.path.join(OUT, "bundle_dense55")
    shutil.rmtree(d, ignore_errors=True)
    RA.save_avatar_bundle(b, d)
    got = RA.load_avatar_bundle(d)
    c = got.canonical
    for k in ("positions", "sh_coeffs", "opacities", "log_scales", "rotations"):
        expected[f"dense55_{k}"] = getattr(c, k)
    expected["dense55_weights"] = got.lbs_weights
    expected["dense55_inv_bind"] = got.inv_bind
    expected["dense55_traj_quats"] = got.trajectory.quats
    expected["dense55_traj_trans"] = got.trajectory.trans
    expected["dense55_fps"] = np.array(got.trajectory.fps)
    # bundles the reference rejects; each file is edited after save_avatar_bundle
    small = S.make_dense_avatar(60, 24, seed=8, sh_degree=0)
    base = to_ref(small, RR.bake_capsules(RA.Skeleton(np.asarray(small.skeleton.parents),
                                                      np.asarray(small.skeleton.rest_positions)),
                                          RA.Trajectory(small.trajectory.fps, np.asarray(small.trajectory.quats),
                                                        np.asarray(small.trajectory.trans))))

    def poke(name, blob, index, value):
        d = os.path.join(OUT, name)
        shutil.rmtree(d, ignore_errors=True)
        RA.save_avatar_bundle(base, d)
        p = os.path.join(d, blob)
        a = np.fromfile(p, dtype="<f4")
        a[index] = value
        a.tofile(p)
        try:
            RA.load_avatar_bundle(d)
            msg = ""
        except Exception as e:  # the reference's exception, compared verbatim
            msg = f"{type(e).__name__}: {e}"
        assert msg, name
        expected[f"{name}_message"] = np.array(msg)

    poke("bad_traj_nan", "trajectory.f32", 5 * 25 * 7 + 3 * 7 + 5, np.nan)
    poke("bad_inv_bind_inf", "inv_bind.f32", 7 * 16 + 3, np.inf)
    poke("bad_capsule_nan", "capsules.f32", 2 * 23 * 7 + 4 * 7 + 1, np.nan)
    poke("bad_capsule_radius", "capsules.f32", 1 * 23 * 7 + 9 * 7 + 6, -0.01)
    np.savez_compressed(os.path.join(OUT, "expected_dense.npz"), **expected)
    for k, v in expected.items():
        if k.endswith("_message"):
            print(k, v)


if __name__ == "__main__":
    gen_lbs()
    gen_bundles()
