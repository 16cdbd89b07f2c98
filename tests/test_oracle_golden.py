"""Pins the CPU oracle (oracle/splat_oracle.c) to the reference's own outputs.

The fixtures in tests/golden/ were produced by tests/golden/make_golden.py, which runs the
reference package and its compiled Cython blend kernel in the build container. The discrete
outputs must match exactly: ids in depth order, the tile CSR, contributor/visited counts and
RenderStats. Continuous outputs must match to within the ulp-level gap between numpy's SIMD exp
and libm's exp.
"""

import hashlib
import math

import numpy as np
import pytest

from conftest import load_cases
from oracle import oracle as O
from paper_2604_12626_b200 import synthetic as S

CONT_TOL = 1e-12


def _digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _check_render_case(case, cloud, cam):
    bg = case.background()
    proj = O.project_cloud(cloud, cam)
    np.testing.assert_array_equal(proj.ids, case["ids"])
    np.testing.assert_array_equal(proj.depths, case["depths"])
    assert [proj.stats[k] for k in ("n_input", "n_culled_depth", "n_culled_frame", "n_degenerate", "n_drawn")] \
        == case["stats"].tolist()
    if "means2d" in case:
        np.testing.assert_array_equal(proj.means2d, case["means2d"])
        for k in ("conics", "colors", "alphas", "radii"):
            ref = case[k]
            if ref.size:
                err = np.abs(getattr(proj, k) - ref).max() / max(np.abs(ref).max(), 1e-300)
                assert err < CONT_TOL, (k, err)
    tiles_x, tiles_y = O.tiles_for(cam.width, cam.height)
    ts, ps = O.bin_tiles(proj.means2d, proj.radii, tiles_x, tiles_y)
    np.testing.assert_array_equal(ts, case["tile_starts"])
    assert ps.size == int(case["n_pairs"])
    if "pair_splat" in case:
        np.testing.assert_array_equal(ps, case["pair_splat"])
    assert _digest(ps.astype(np.int32)) == str(case["pairs_digest"])
    fr = O.rasterize(cloud, cam, bg)
    np.testing.assert_array_equal(fr.contrib, case["contrib"].astype(np.int32))
    np.testing.assert_array_equal(fr.visited, case["visited"].astype(np.int32))
    tol = CONT_TOL if case["color"].dtype == np.float64 else 1e-6
    assert np.abs(fr.color - case["color"]).max() < tol
    assert np.abs(fr.depth - case["depth"]).max() < tol * 100
    if "alpha" in case:
        assert np.abs(fr.alpha - case["alpha"]).max() < tol
    brute = O.rasterize_reference(cloud, cam, bg)
    assert np.array_equal(brute.color, fr.color) and np.array_equal(brute.contrib, fr.contrib)


@pytest.mark.parametrize("name", ["c1_scenes", "edges"])
def test_oracle_matches_reference_small(name):
    for case in load_cases(name):
        _check_render_case(case, case.cloud(), case.camera())


def test_oracle_matches_reference_config0():
    (case,) = load_cases("config0")
    scene, cam = S.config0()
    arrays = [scene.positions, scene.sh_coeffs, scene.opacities, scene.log_scales, scene.rotations]
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(case["input_digest"]), "synthetic config-0 generator drifted"
    _check_render_case(case, scene, cam)


def test_oracle_matches_reference_room():
    cases = load_cases("room")
    box = S.room_box(1_000_000)
    scene = S.make_scene(100_000, box[0], box[1], seed=5)
    cams = S.room_cameras(2, box, seed=6)
    for case, cam in zip(cases, cams):
        _check_render_case(case, scene, cam)


def test_oracle_lbs_and_sample_pose_match_reference():
    for case in load_cases("lbs"):
        q, t = O.sample_pose(case["traj_quats"], case["traj_trans"], float(case["fps"]), float(case["t"]))
        np.testing.assert_array_equal(q, case["pose_quats"])
        np.testing.assert_array_equal(t, case["pose_trans"])
        pos, rot = O.lbs_deform(case["canon_positions"], case["canon_rotations"], case["weights"], case["inv_bind"],
                                q, t)
        assert np.abs(pos - case["out_positions"]).max() <= 1e-12
        assert np.abs(rot - case["out_rotations"]).max() <= 1e-12


def test_oracle_render_observation_matches_reference():
    for case in load_cases("observation"):
        scene = case.cloud("scene_")
        avatars = [case.cloud(f"avatar{i}_") for i in range(int(case["n_avatars"]))]
        out = O.render_observation(scene, avatars, case.camera(), case["background"])
        assert np.abs(out.color - case["color"]).max() < CONT_TOL
        assert np.abs(out.depth - case["depth"]).max() < CONT_TOL * 100
        assert np.abs(out.alpha - case["alpha"]).max() < CONT_TOL
        if avatars:
            assert np.abs(out.layer.color - case["layer_color"]).max() < CONT_TOL


def test_oracle_sample_pose_rejects_negative_time():
    case = load_cases("lbs")[0]
    with pytest.raises(ValueError):
        O.sample_pose(case["traj_quats"], case["traj_trans"], 30.0, -0.1)


def test_oracle_threaded_batch_equals_serial():
    box = S.room_box(1_000_000)
    scene = S.make_scene(20_000, box[0], box[1], seed=3)
    cams = S.room_cameras(3, box, seed=4, width=96, height=64)
    c, a, d = O.render_batch(scene, None, cams, np.array([1.0, 1.0, 1.0]), threads=3)
    for e, cam in enumerate(cams):
        fr = O.rasterize(scene, cam, np.array([1.0, 1.0, 1.0]), counters=False)
        assert np.array_equal(fr.color, c[e]) and np.array_equal(fr.depth, d[e])
    assert math.isfinite(float(c.sum()))
