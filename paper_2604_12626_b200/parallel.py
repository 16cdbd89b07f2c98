"""Multi-GPU plumbing: one process per GPU, environments sharded in contiguous blocks.

Environments are independent (no exchange in the render), so each rank renders its block of
envs against its own replica of the scene and avatar set. The only collective is the optional
gather of quantized observations to rank 0 (uint8 RGB + fp16 depth), done with
torch.distributed (NCCL over NVLink/NVSwitch on GPUs; gloo in CPU tests).
"""

import torch
import torch.distributed as dist


def env_shard(n_envs, world_size, rank):
    """Env e goes to rank floor(e * G / E): contiguous blocks, sizes differ by at most one."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} for world size {world_size}")
    start = -(-rank * n_envs // world_size)
    stop = -(-(rank + 1) * n_envs // world_size)
    return start, stop


def rank_of_env(e, n_envs, world_size):
    return (e * world_size) // n_envs


def gather_observations(rgb, depth, n_envs, dst=0, group=None):
    """Gather every rank's (E_r,H,W,3) uint8 rgb and (E_r,H,W) fp16 depth to rank `dst`.

    Returns (rgb_all, depth_all) on dst (ordered by env id), (None, None) elsewhere. Ranks hold
    env_shard blocks, so concatenating in rank order restores env order. Blocks can differ in
    size by one env; they are padded to the largest block for the collective.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [env_shard(n_envs, world, r) for r in range(world)]
    counts = [b - a for a, b in sizes]
    cap = max(counts)
    pad = cap - rgb.shape[0]

    def padded(t):
        if pad == 0:
            return t.contiguous()
        return torch.cat([t, t.new_zeros((pad,) + tuple(t.shape[1:]))]).contiguous()

    send_rgb, send_depth = padded(rgb), padded(depth.contiguous().view(torch.uint8))  # fp16 as bytes
    if rank == dst:
        rgb_list = [torch.empty_like(send_rgb) for _ in range(world)]
        depth_list = [torch.empty_like(send_depth) for _ in range(world)]
    else:
        rgb_list = depth_list = None
    dist.gather(send_rgb, rgb_list, dst=dst, group=group)
    dist.gather(send_depth, depth_list, dst=dst, group=group)
    if rank != dst:
        return None, None
    rgb_all = torch.cat([t[:c] for t, c in zip(rgb_list, counts)])
    depth_all = torch.cat([t[:c] for t, c in zip(depth_list, counts)]).view(torch.float16)
    return rgb_all, depth_all


def render_sharded(renderer, cameras, sim_times=None, gather=True, dst=0, group=None):
    """One step of the env-sharded batch: this rank renders its contiguous block
    env_shard(E, G, rank) of the E environments with `renderer` (a batch.BatchRenderer holding its
    own replica of the scene and avatar set), the render's epilogues write the uint8 RGB + fp16 depth
    payload, and -- when `gather` -- the payload of all E envs is gathered to rank `dst` in env order.

    Returns (local, gathered): local = the render_frames dict of this rank's block (float frames +
    payload), gathered = (rgb8 (E,H,W,3), depth16 (E,H,W)) on dst, None elsewhere. With the gloo
    backend (CPU tests) the payload is staged through host memory; NCCL gathers device tensors.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = len(cameras)
    a, b = env_shard(n, world, rank)
    times = None if sim_times is None else list(sim_times)[a:b]
    local = renderer.render(list(cameras)[a:b], times, payload=True)
    if not gather:
        return local, None
    if world == 1:
        return local, (local["rgb8"], local["depth16"])
    rgb, depth = local["rgb8"], local["depth16"]
    if dist.get_backend(group) != "nccl":
        rgb, depth = rgb.cpu(), depth.cpu()
    out = gather_observations(rgb, depth, n, dst=dst, group=group)
    return local, (out if rank == dst else None)
