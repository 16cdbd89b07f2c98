"""CPU tests: the C-ABI library surface, host-side packing/layout logic, env sharding and the
observation gather over a 2-rank gloo group. No GPU compute is called here."""

import ctypes
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO
from paper_2604_12626_b200 import _native as N
from paper_2604_12626_b200 import synthetic as S
from paper_2604_12626_b200.camera import Camera, pose_world_to_camera
from paper_2604_12626_b200.device import CAMERA_DTYPE, sparse_influences
from paper_2604_12626_b200.errors import ContractViolation, ValidationError
from paper_2604_12626_b200.parallel import env_shard, gather_observations, rank_of_env

HEADER = os.path.join(REPO, "include", "splatnav_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2604_12626_b200 import build
    build.build()
    lib = ctypes.CDLL(N.LIB_PATH)
    missing = [s for s in declared_functions() if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(N.EXPORTS) == declared_functions()
    assert N.load().sn_abi_version() == N.ABI_VERSION == 3


def _c_layout(struct, fields):
    """sizeof / offsetof of a header struct, from a C program compiled against the header."""
    import subprocess
    import tempfile
    body = f'printf("%zu", sizeof({struct}));' + "".join(
        f'printf(" %zu", offsetof({struct}, {f}));' for f in fields)
    src = f'#include <stdio.h>\n#include "splatnav_b200.h"\nint main(void) {{ {body} return 0; }}\n'
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "t.c"), os.path.join(d, "t")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-std=c11", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        vals = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    return vals[0], vals[1:]


@pytest.mark.parametrize("cls,struct", [(N.SnCamera, "sn_camera"), (N.SnStats, "sn_stats"), (N.SnCloud, "sn_cloud"),
                                        (N.SnAvatars, "sn_avatars"), (N.SnRenderOpts, "sn_render_opts")])
def test_struct_layouts_match_header(cls, struct):
    """The ctypes mirrors have the C compiler's size and field offsets for every header struct."""
    names = [f[0] for f in cls._fields_]
    size, offs = _c_layout(struct, names)
    assert ctypes.sizeof(cls) == size
    assert [getattr(cls, f).offset for f in names] == offs
    if cls is N.SnCamera:
        assert size == CAMERA_DTYPE.itemsize


def test_camera_array_packs_reference_centre():
    from paper_2604_12626_b200.device import camera_array
    w2c = pose_world_to_camera(np.array([1.0, 2.0, 1.25]), 0.7)
    cam = Camera.from_hfov(640, 480, 90.0, 0.1, 100.0, w2c)
    buf = camera_array([cam], np.array([0.1, 0.2, 0.3]))
    c = buf[0]
    assert (c.fx, c.cx, c.cy, c.width, c.height, c.has_background) == (cam.fx, 320.0, 240.0, 640, 480, 1)
    np.testing.assert_array_equal(np.array(c.center[:]), cam.center)
    np.testing.assert_array_equal(np.array(c.rot[:]).reshape(3, 3), w2c[:3, :3])
    assert camera_array([cam], None)[0].has_background == 0


def test_sparse_influences_roundtrip_and_order():
    rng = np.random.default_rng(0)
    n, j = 200, 24
    dense = np.zeros((n, j))
    for i in range(n):
        js = rng.choice(j, size=rng.integers(1, 5), replace=False)
        dense[i, js] = rng.dirichlet(np.ones(js.size))
    packed, w = sparse_influences(dense)
    back = np.zeros_like(dense)
    for i in range(n):
        jj = [(int(packed[i]) >> (8 * k)) & 0xFF for k in range(4)]
        nz = [k for k in range(4) if w[i, k] != 0.0]
        assert [jj[k] for k in nz] == sorted(jj[k] for k in nz)  # ascending joint order
        for k in nz:
            back[i, jj[k]] = w[i, k]
    np.testing.assert_array_equal(back, dense)


def test_sparse_influences_rejects_more_than_four():
    dense = np.full((3, 6), 1.0 / 6)
    with pytest.raises(ContractViolation):
        sparse_influences(dense)


def test_env_shard_partitions_contiguously():
    for n_envs in (1, 7, 64, 1024):
        for world in (1, 2, 3, 8):
            covered = []
            for r in range(world):
                a, b = env_shard(n_envs, world, r)
                covered.extend(range(a, b))
                for e in range(a, b):
                    assert rank_of_env(e, n_envs, world) == r
            assert covered == list(range(n_envs))
            sizes = [np.subtract(*env_shard(n_envs, world, r)[::-1]) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, n_envs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = env_shard(n_envs, world, rank)
    h, w = 3, 5
    env_ids = torch.arange(a, b, dtype=torch.int64)
    rgb = (env_ids.view(-1, 1, 1, 1) * 7 + torch.arange(h * w * 3).view(1, h, w, 3)).remainder(256).to(torch.uint8)
    depth = (env_ids.view(-1, 1, 1).double() + torch.linspace(0, 1, h * w).view(1, h, w)).to(torch.float16)
    rgb_all, depth_all = gather_observations(rgb, depth, n_envs, dst=0)
    if rank == 0:
        q.put((rgb_all.numpy(), depth_all.float().numpy()))
    dist.destroy_process_group()


def test_gather_observations_two_ranks_gloo():
    n_envs, world = 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n_envs, q)) for r in range(world)]
    for p in procs:
        p.start()
    rgb_all, depth_all = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    h, w = 3, 5
    env_ids = np.arange(n_envs)
    want_rgb = ((env_ids.reshape(-1, 1, 1, 1) * 7 + np.arange(h * w * 3).reshape(1, h, w, 3)) % 256).astype(np.uint8)
    np.testing.assert_array_equal(rgb_all, want_rgb)
    want_depth = (env_ids.reshape(-1, 1, 1) + np.linspace(0, 1, h * w).reshape(1, h, w)).astype(np.float16)
    np.testing.assert_array_equal(depth_all, want_depth.astype(np.float32))


def test_raster_registry_contract(monkeypatch):
    from paper_2604_12626_b200 import raster
    assert sorted(raster.available_kernels()) == ["cuda"]
    assert raster.get_kernel().KERNEL_NAME == "cuda"
    with pytest.raises(ValueError):
        raster.get_kernel("cython")
    monkeypatch.setenv("SPLATNAV_KERNEL", "python")
    with pytest.raises(ValueError):
        raster.get_kernel()


def test_synthetic_config_shapes_and_determinism():
    a = S.make_scene(1000, [0, 0, 0], [8, 8, 3], seed=3)
    b = S.make_scene(1000, [0, 0, 0], [8, 8, 3], seed=3)
    assert a.positions.dtype == np.float32 and a.sh_coeffs.shape == (1000, 16, 3)
    assert a.positions.tobytes() == b.positions.tobytes()
    av = S.make_avatar(2000, seed=1, n_frames=4)
    assert av.lbs_weights.shape == (2000, 24)
    assert ((av.lbs_weights > 0).sum(axis=1) == 4).all()
    np.testing.assert_allclose(av.lbs_weights.sum(axis=1), 1.0, atol=1e-6)
    assert av.trajectory.quats.shape == (4, 25, 4)
    lo, hi = S.room_box(6_000_000)
    assert np.isclose(hi[0] * hi[1] * hi[2], 8 * 8 * 3 * 6)


def test_containers_validate_like_reference():
    with pytest.raises(ValidationError):
        Camera(0.0, 1.0, 0, 0, 4, 4, 0.1, 10.0, np.eye(4))
    with pytest.raises(ValidationError):
        Camera(1.0, 1.0, 0, 0, 4, 4, 1.0, 0.5, np.eye(4))
    c = S.make_scene(10, [0, 0, 0], [1, 1, 1], seed=0)
    c.rotations = c.rotations * 2.0
    c.validate()
    np.testing.assert_allclose(np.linalg.norm(c.rotations, axis=1), 1.0, atol=1e-6)
    c.positions[0, 0] = np.nan
    with pytest.raises(ValidationError):
        c.validate()
