"""Asset ingest: PLY and avatar-bundle directories unpacked on the device
must equal what the reference's loaders (splatnav.ply.load_gaussian_ply, splatnav.avatar.
load_avatar_bundle) produce for the same files -- bit for bit, including the float32 quaternion
renormalization and the float64 weight renormalization. Fixtures: tests/golden/assets/, written and
read back by the reference itself (tests/golden/make_assets.py)."""

import os

import numpy as np
import pytest
import torch

from conftest import REPO
from paper_2604_12626_b200 import assets as A
from paper_2604_12626_b200.errors import PlyParseError, UnsupportedLayoutError, ValidationError

D = os.path.join(REPO, "tests", "golden", "assets")
E = np.load(os.path.join(D, "expected.npz"))


def _write_ply(path, header_lines, payload=b""):
    with open(path, "wb") as f:
        f.write(("\n".join(header_lines) + "\n").encode("ascii"))
        f.write(payload)


# ---------------------------------------------------------------- host side (no GPU)

def test_ply_header_errors_match_reference(tmp_path):
    p = str(tmp_path / "x.ply")
    _write_ply(p, ["ply", "format ascii 1.0", "end_header"])
    with pytest.raises(PlyParseError, match="unsupported format line 'format ascii 1.0'"):
        A.read_ply_table(p)
    _write_ply(p, ["ply", "format binary_little_endian 1.0", "element vertex 2", "property float x",
                   "end_header"], b"\0" * 4)
    with pytest.raises(PlyParseError, match="payload truncated: expected 8 bytes, got 4"):
        A.read_ply_table(p)
    _write_ply(p, ["ply", "format binary_little_endian 1.0", "element vertex 1", "property float x",
                   "end_header"], b"\0" * 4)
    with pytest.raises(UnsupportedLayoutError, match="missing required properties"):
        A.read_ply_table(p)
    _write_ply(p, ["ply", "format binary_little_endian 1.0", "element vertex 1", "property double x",
                   "end_header"])
    with pytest.raises(PlyParseError, match="only float32 is handled"):
        A.read_ply_table(p)


def test_ply_column_map_follows_the_header():
    table, cols, k = A.read_ply_table(os.path.join(D, "scene_deg1_permuted.ply"))
    assert k == 4 and table.shape == (333, 26)
    # x y z f_dc_0..2 opacity scale_0..2 rot_0..3 f_rest_0..8 in the file's column numbering
    assert cols.tolist() == [0, 1, 2, 11, 12, 13, 10, 14, 15, 16, 6, 7, 8, 9] + list(range(17, 26))


# ---------------------------------------------------------------- device unpack (GPU)

@pytest.mark.gpu
@pytest.mark.parametrize("name,prefix", [("scene_deg3.ply", "deg3"), ("scene_deg1_permuted.ply", "deg1")])
def test_ply_unpacks_like_reference(name, prefix):
    dc = A.load_gaussian_ply(os.path.join(D, name))
    pos, sh, op, ls, rot = dc.to_host()
    np.testing.assert_array_equal(pos, E[f"{prefix}_positions"])
    np.testing.assert_array_equal(sh, E[f"{prefix}_sh_coeffs"])
    np.testing.assert_array_equal(op, E[f"{prefix}_opacities"])
    np.testing.assert_array_equal(ls, E[f"{prefix}_log_scales"])
    np.testing.assert_array_equal(rot, E[f"{prefix}_rotations"])  # float32 renormalization, bit-exact


@pytest.mark.gpu
def test_ply_nonfinite_raises_reference_message():
    with pytest.raises(ValidationError) as ei:
        A.load_gaussian_ply(os.path.join(D, "scene_nonfinite.ply"))
    assert f"ValidationError: {ei.value}" == str(E["nonfinite_message"])


@pytest.mark.gpu
def test_bundles_unpack_like_reference():
    from paper_2604_12626_b200.device import DeviceAvatars, sparse_influences
    dav = A.load_avatar_bundles([os.path.join(D, "bundle_a"), os.path.join(D, "bundle_b")],
                                start_offsets=[0.0, 0.3], loops=[1, 0])
    assert dav.counts == [300, 200] and dav.sh_k == 9 and dav.n_joints == 11
    po = dav.pos_opacity.cpu().numpy()
    sh = dav.sh.cpu().numpy()
    rows = {"bundle_a": slice(0, 300), "bundle_b": slice(300, 500)}
    for name, r in rows.items():
        np.testing.assert_array_equal(po[r, :3], E[f"{name}_positions"].astype(np.float64))
        np.testing.assert_array_equal(po[r, 3], E[f"{name}_opacities"].astype(np.float64))
        np.testing.assert_array_equal(dav.log_scales.cpu().numpy()[r, :3], E[f"{name}_log_scales"])
        np.testing.assert_array_equal(dav.rotations.cpu().numpy()[r], E[f"{name}_rotations"].astype(np.float64))
        shr = E[f"{name}_sh_coeffs"]
        k = shr.shape[1]
        np.testing.assert_array_equal(sh[:3 * k, r].T.reshape(-1, k, 3), shr)
        assert not sh[3 * k:, r].any()  # concat_clouds zero-pads SH (cloud.py:110-129)
        jpk, wts = sparse_influences(E[f"{name}_weights"])  # weights renormalized like the reference
        np.testing.assert_array_equal(dav.joints.cpu().numpy()[r].view(np.uint32), jpk)
        np.testing.assert_array_equal(dav.weights.cpu().numpy()[r], wts)
    # the same set packed on the host from the reference-loaded bundles: identical device buffers
    class B:
        pass
    bundles = []
    for name in rows:
        b = B()
        b.canonical = B()
        b.canonical.positions = E[f"{name}_positions"]
        b.canonical.opacities = E[f"{name}_opacities"]
        b.canonical.log_scales = E[f"{name}_log_scales"]
        b.canonical.rotations = E[f"{name}_rotations"]
        b.canonical.sh_coeffs = E[f"{name}_sh_coeffs"]
        b.lbs_weights = E[f"{name}_weights"]
        b.inv_bind = E[f"{name}_inv_bind"]
        b.trajectory = B()
        b.trajectory.quats = E[f"{name}_traj_quats"]
        b.trajectory.trans = E[f"{name}_traj_trans"]
        b.trajectory.fps = float(E[f"{name}_fps"])
        bundles.append(b)
    host = DeviceAvatars(bundles, start_offsets=[0.0, 0.3], loops=[1, 0])
    for attr in ("pos_opacity", "log_scales", "rotations", "sh", "joints", "weights", "avatar_of", "inv_bind",
                 "traj_q", "traj_t", "traj_offset", "n_frames", "fps", "start_offset", "loop"):
        assert torch.equal(getattr(dav, attr), getattr(host, attr)), attr


@pytest.mark.gpu
def test_render_from_loaded_ply_equals_host_packed_cloud():
    from paper_2604_12626_b200 import renderer, synthetic as S
    from paper_2604_12626_b200.device import DeviceCloud
    dc = A.load_gaussian_ply(os.path.join(D, "scene_deg3.ply"))

    class C:
        pass
    c = C()
    c.positions, c.sh_coeffs, c.opacities = E["deg3_positions"], E["deg3_sh_coeffs"], E["deg3_opacities"]
    c.log_scales, c.rotations = E["deg3_log_scales"], E["deg3_rotations"]
    host = DeviceCloud(c)
    cams = S.room_cameras(2, (np.array([-5.0, -5.0, -4.0]), np.array([5.0, 5.0, 6.0])), seed=5, width=160, height=120)
    a = renderer.render_frames(dc, cams, np.ones(3), contrib=True)
    b = renderer.render_frames(host, cams, np.ones(3), contrib=True)
    for k in ("color", "alpha", "depth", "contrib_scene"):
        assert torch.equal(a[k], b[k]), k
