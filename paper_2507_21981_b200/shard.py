"""Multi-GPU plumbing: environment sharding and the frame gather of BASELINE config 4.

Every (environment, camera) render is independent given the replicated background, so the
render path shards by environment with no data-path collective. The only real
exchange is config 4's gather of finished frames to rank 0, done here with torch.distributed
point-to-point (NCCL over NVLink on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def env_range(n_envs: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split of n_envs environments over world ranks: [begin, end)."""
    base, extra = divmod(n_envs, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def env_chunks(begin: int, end: int, chunk: int = 64):
    """Launch-sized chunks (config 2 size) of a rank's environments."""
    for b in range(begin, end, chunk):
        yield b, min(end, b + chunk)


def gather_frames(frames: torch.Tensor, n_envs: int, floats_per_env: int, dst: int = 0):
    """Gather every rank's frames (its env_range, env-major, floats_per_env floats each) to
    rank `dst`, which returns the full [n_envs * floats_per_env] tensor in environment order;
    other ranks return None. Grouped point-to-point sends, one per rank (NCCL has no gather)."""
    rank, world = dist.get_rank(), dist.get_world_size()
    if rank != dst:
        dist.send(frames.contiguous(), dst=dst)
        return None
    out = torch.empty(n_envs * floats_per_env, dtype=frames.dtype, device=frames.device)
    reqs = []
    for r in range(world):
        b, e = env_range(n_envs, r, world)
        view = out[b * floats_per_env: e * floats_per_env]
        if r == dst:
            view.copy_(frames)
        elif e > b:
            reqs.append(dist.irecv(view, src=r))
    for q in reqs:
        q.wait()
    return out


def max_over_ranks(value: float, device) -> float:
    """Max of a per-rank scalar (device time) over all ranks."""
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
