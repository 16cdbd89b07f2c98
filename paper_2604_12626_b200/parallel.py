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
