"""Multi-GPU plumbing: rank launch, env sharding and the statistics all-reduce
(SURVEY §8(e)).

The step has no exchange at all: rank g of G owns its own batch of envs (weak
scaling, envs_per_rank fixed), and the only collective is one all-reduce of a
few scalars after a rollout — the analogue of the paper's normalisation
statistics "synced between all cores".  Backend-agnostic:
NCCL on GPUs, gloo in the CPU tests, which run these same functions.
"""
from __future__ import annotations

import os
import socket
import subprocess
import sys
from dataclasses import dataclass


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


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_or_check(gpus: int, script: str, argv: list[str]) -> int | None:
    """One process per GPU.  Under a launcher (WORLD_SIZE set) check that it started
    exactly `gpus` ranks and return None (the caller continues as that rank).  Without
    one and gpus > 1, start `gpus` ranks of `script argv` with torch.distributed.run on
    127.0.0.1 and return their exit code (the caller exits with it)."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != gpus:
            raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={ws}: launch one rank per GPU")
        return None
    if gpus <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", script, *argv]
    return subprocess.call(cmd)


@dataclass
class Ranks:
    rank: int
    world: int
    local: int
    backend: str | None      # None for a single process without a process group
    nranks: int              # the communicator's size as the process group reports it


def init_ranks(backend: str) -> Ranks:
    """Read RANK / WORLD_SIZE / LOCAL_RANK (torchrun), bind the local GPU for "nccl", and
    create the process group for world > 1 or any torchrun launch (a one-rank communicator
    at N = 1, so the launcher's path is the one exercised).  Logs the communicator size."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend == "nccl":
        torch.cuda.set_device(local)
    if world == 1 and "TORCHELASTIC_RUN_ID" not in os.environ:
        return Ranks(rank, 1, local, None, 1)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    n = dist.get_world_size()
    if n != world:
        raise SystemExit(f"process group has {n} ranks, WORLD_SIZE={world}")
    print(f"[rank {rank}/{world}] {backend} communicator: nranks={n}", file=sys.stderr, flush=True)
    return Ranks(rank, world, local, backend, n)


def barrier(r: Ranks) -> None:
    if r.backend is not None:
        import torch.distributed as dist
        dist.barrier()


def allreduce_stats(env_steps: float, blowups: float, elapsed_ms: float, return_sum: float = 0.0, device=None):
    """SUM of [env_steps, blowups, return_sum] and MAX of [elapsed_ms] over ranks (≤ 32 B each way).

    Returns (env_steps, blowups, return_sum, elapsed_ms_max) as Python floats."""
    import torch
    import torch.distributed as dist
    s = torch.tensor([env_steps, blowups, return_sum], dtype=torch.float64, device=device)
    m = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
    return float(s[0]), float(s[1]), float(s[2]), float(m[0])


def allreduce_max(x: float, device=None) -> float:
    """MAX over ranks of one timing (ms); identity for a single process."""
    return allreduce_stats(0.0, 0.0, x, device=device)[3]


def finalize(r: Ranks) -> None:
    if r.backend is not None:
        import torch.distributed as dist
        dist.destroy_process_group()
