"""Multi-GPU plumbing: env sharding and the statistics all-reduce.

The step has no exchange at all: rank g of G owns its own batch of envs (weak
scaling, envs_per_rank fixed), and the only collective is one all-reduce of a
few scalars after a rollout — the analogue of the paper's normalisation
statistics "synced between all cores".  Backend-agnostic
(NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations


def env_shard(rank: int, world: int, envs_per_rank: int):
    """Global env index range [start, stop) owned by `rank` under weak scaling."""
    if not (0 <= rank < world) or envs_per_rank < 0:
        raise ValueError("bad rank/world/envs_per_rank")
    start = rank * envs_per_rank
    return start, start + envs_per_rank


def strong_shard(rank: int, world: int, n_total: int):
    """[start, stop) for a fixed total (strong scaling): contiguous, sizes differ by ≤ 1."""
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def allreduce_stats(env_steps: float, blowups: float, elapsed_ms: float, return_sum: float = 0.0, device=None):
    """SUM of [env_steps, blowups, return_sum] and MAX of [elapsed_ms] over ranks (≤ 32 B each way).

    Returns (env_steps, blowups, return_sum, elapsed_ms_max) as Python floats."""
    import torch
    import torch.distributed as dist
    s = torch.tensor([env_steps, blowups, return_sum], dtype=torch.float64, device=device)
    m = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
    return float(s[0]), float(s[1]), float(s[2]), float(m[0])
