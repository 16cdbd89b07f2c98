"""Generates the asset-ingest fixtures under tests/golden/assets/ with the REFERENCE package's own
writers and readers (splatnav.ply / splatnav.avatar, /root/reference/pkg/src), run in the build
container only. The GPU tests load the same files through assets.py (device unpack) and compare
with the arrays the reference's loaders produced.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_assets.py
"""
import json
import os
import shutil
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from splatnav import avatar as RA  # noqa: E402
from splatnav import ply as RP  # noqa: E402
from splatnav import synthetic as RS  # noqa: E402
from splatnav.cloud import GaussianCloud  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "assets")


def cloud_arrays(c):
    return {"positions": c.positions, "sh_coeffs": c.sh_coeffs, "opacities": c.opacities,
            "log_scales": c.log_scales, "rotations": c.rotations}


def main():
    if os.path.isdir(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    expected = {}
    # 1. degree-3 cloud whose quaternions are off unit norm (the float32 renormalization runs)
    c = RS.random_cloud(700, seed=11, sh_degree=3)
    rng = np.random.default_rng(12)
    c.rotations = (c.rotations * rng.uniform(0.5, 2.0, size=(700, 1))).astype(np.float32)
    RP.save_gaussian_ply(c, os.path.join(OUT, "scene_deg3.ply"))
    got = RP.load_gaussian_ply(os.path.join(OUT, "scene_deg3.ply"))
    expected.update({f"deg3_{k}": v for k, v in cloud_arrays(got).items()})
    # 2. degree-1 cloud in a hand-written header: normals, comments, permuted properties
    c1 = RS.random_cloud(333, seed=13, sh_degree=1)
    names = ["x", "y", "z", "nx", "ny", "nz", "rot_0", "rot_1", "rot_2", "rot_3", "opacity",
             "f_dc_0", "f_dc_1", "f_dc_2", "scale_0", "scale_1", "scale_2"] + [f"f_rest_{i}" for i in range(9)]
    n = c1.n
    cols = {"x": c1.positions[:, 0], "y": c1.positions[:, 1], "z": c1.positions[:, 2],
            "nx": np.zeros(n), "ny": np.ones(n), "nz": np.zeros(n), "opacity": c1.opacities}
    for i in range(4):
        cols[f"rot_{i}"] = c1.rotations[:, i]
    for i in range(3):
        cols[f"f_dc_{i}"] = c1.sh_coeffs[:, 0, i]
        cols[f"scale_{i}"] = c1.log_scales[:, i]
    rest = c1.sh_coeffs[:, 1:, :].transpose(0, 2, 1).reshape(n, 9)  # channel-major on disk
    for i in range(9):
        cols[f"f_rest_{i}"] = rest[:, i]
    table = np.stack([np.asarray(cols[k], dtype="<f4") for k in names], axis=1)
    header = "ply\nformat binary_little_endian 1.0\ncomment written by make_assets.py\n"
    header += f"element vertex {n}\n" + "".join(f"property float {k}\n" for k in names)
    header += "element face 0\nproperty list uchar int vertex_indices\nend_header\n"
    with open(os.path.join(OUT, "scene_deg1_permuted.ply"), "wb") as f:
        f.write(header.encode("ascii"))
        f.write(table.tobytes())
    got = RP.load_gaussian_ply(os.path.join(OUT, "scene_deg1_permuted.ply"))
    expected.update({f"deg1_{k}": v for k, v in cloud_arrays(got).items()})
    # 3. non-finite log-scales: the reference's ValidationError message
    c2 = RS.random_cloud(50, seed=14, sh_degree=0)
    ls = c2.log_scales.copy()
    ls[3, 1] = np.nan
    ls[7, 0] = np.inf
    bad = GaussianCloud(c2.positions, c2.sh_coeffs, c2.opacities, c2.log_scales, c2.rotations)
    RP.save_gaussian_ply(bad, os.path.join(OUT, "scene_nonfinite.ply"))
    raw = open(os.path.join(OUT, "scene_nonfinite.ply"), "rb").read()
    hdr_end = raw.index(b"end_header\n") + len(b"end_header\n")
    tab = np.frombuffer(raw[hdr_end:], dtype="<f4").reshape(50, -1).copy()
    tab[:, -7:-4] = ls
    open(os.path.join(OUT, "scene_nonfinite.ply"), "wb").write(raw[:hdr_end] + tab.tobytes())
    try:
        RP.load_gaussian_ply(os.path.join(OUT, "scene_nonfinite.ply"))
        msg = ""
    except Exception as e:  # the reference's message, compared verbatim
        msg = f"{type(e).__name__}: {e}"
    expected["nonfinite_message"] = np.array(msg)
    # 4./5. avatar bundles: degree 2 with weight rows off by 5e-5 (renormalized), degree 0
    for name, seed, deg, scale in (("bundle_a", 21, 2, 1.00005), ("bundle_b", 22, 0, 1.0)):
        b = RS.make_avatar_bundle(n_gaussians=300 if deg else 200, seed=seed, sh_degree=deg)
        if deg:
            sh = np.asarray(b.canonical.sh_coeffs).copy()
            sh[:, 1:, :] = np.random.default_rng(seed).normal(0, 0.05, size=sh[:, 1:, :].shape)
            b.canonical.sh_coeffs = sh.astype(np.float32)
        b.lbs_weights = b.lbs_weights * scale
        d = os.path.join(OUT, name)
        RA.save_avatar_bundle(b, d)
        got = RA.load_avatar_bundle(d)
        for k, v in cloud_arrays(got.canonical).items():
            expected[f"{name}_{k}"] = v
        expected[f"{name}_weights"] = got.lbs_weights
        expected[f"{name}_inv_bind"] = got.inv_bind
        expected[f"{name}_traj_quats"] = got.trajectory.quats
        expected[f"{name}_traj_trans"] = got.trajectory.trans
        expected[f"{name}_fps"] = np.array(got.trajectory.fps)
    np.savez_compressed(os.path.join(OUT, "expected.npz"), **expected)
    print(json.dumps({k: list(np.shape(v)) for k, v in expected.items()}, indent=0))


if __name__ == "__main__":
    main()
