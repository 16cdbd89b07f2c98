"""Env sharding as an execution path: the observation payload written by the
render's epilogues equals sn_quantize_frames of the float frames (frame_io's rule), and a batch
rendered as 2 ranks (2 processes, gloo, each on cuda:0 with its own replica) and gathered to rank 0
is bit-identical to the same batch rendered by one process. The ranks share one GPU here (the pool
gives one per call); they never wait on each other's kernels -- the only exchange is the gather."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(n_envs=7):
    from paper_2604_12626_b200 import synthetic as S
    box = S.room_box(1_000_000)
    scene = S.make_scene(40_000, box[0], box[1], seed=121)
    bundles = [S.make_avatar(3000, seed=122 + i, n_frames=12, floor_lo=(2.0, 2.0), floor_hi=(6.0, 6.0))
               for i in range(2)]
    cams = S.room_cameras(n_envs, box, seed=123, width=96, height=64)
    times = np.linspace(0.0, 0.37, n_envs)
    return scene, bundles, cams, times


def test_payload_equals_quantized_frames():
    from paper_2604_12626_b200.batch import BatchRenderer
    from paper_2604_12626_b200.frame_io import quantize
    scene, bundles, cams, times = _setup()
    for exact in (False, True):
        br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.2], background=(0.3, 0.6, 0.9))
        out = br.render(cams, times, payload=True, exact=exact)
        rgb, d16 = quantize(out["color"], out["depth"])
        assert torch.equal(out["rgb8"], rgb)
        assert torch.equal(out["depth16"].view(torch.int16), d16.view(torch.int16))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_12626_b200.batch import BatchRenderer
    from paper_2604_12626_b200.parallel import render_sharded
    scene, bundles, cams, times = _setup()
    br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.2], background=(0.3, 0.6, 0.9))
    local, gathered = render_sharded(br, cams, times)
    if rank == 0:
        q.put((gathered[0].cpu().numpy(), gathered[1].view(torch.int16).cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_render_equals_one_process():
    import torch.multiprocessing as mp
    from paper_2604_12626_b200.batch import BatchRenderer
    scene, bundles, cams, times = _setup()
    br = BatchRenderer(scene, bundles, start_offsets=[0.0, 0.2], background=(0.3, 0.6, 0.9))
    ref = br.render(cams, times, payload=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    rgb, d16 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_array_equal(rgb, ref["rgb8"].cpu().numpy())
    np.testing.assert_array_equal(d16, ref["depth16"].view(torch.int16).cpu().numpy())
