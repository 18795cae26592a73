"""World-size-2 gloo tests of the N>1 host path (CPU): env sharding, the
statistics all-reduce, and that sharded stepping reproduces the unsharded
result exactly (envs are independent)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2106_13281_b200.dist import env_shard, strong_shard


def test_shard_ranges_cover_exactly():
    for world in (1, 2, 3, 8):
        for n in (0, 1, 7, 8192, 8193):
            spans = [strong_shard(r, world, n) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
        assert [env_shard(r, world, 8192) for r in range(world)] == [(r * 8192, (r + 1) * 8192) for r in range(world)]
    with pytest.raises(ValueError):
        env_shard(2, 2, 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    import oracle
    import synth
    from paper_2106_13281_b200.dist import allreduce_stats, strong_shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = oracle.Oracle(oracle.load_scene("ant"))
    qp = o.reset(n_total, 3, 0.1, 0.1)
    acts = synth.actions(4, 3, n_total, o.act_dim)
    lo, hi = strong_shard(rank, world, n_total)
    mine = {k: v[lo:hi] for k, v in qp.items()}
    blow = 0
    for t in range(3):
        mine, ex = o.step(mine, acts[t][lo:hi])
        blow += int((ex["status"] != 0).sum())
    steps, blowups, _, ms = allreduce_stats(float((hi - lo) * 3), float(blow), float(10 + rank))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), lo=lo, hi=hi, steps=steps, blowups=blowups, ms=ms,
             **{k: v for k, v in mine.items()})
    dist.destroy_process_group()


def test_gloo_world2_sharded_equals_unsharded(tmp_path):
    import oracle
    import synth
    n_total, world = 77, 2
    mp.start_processes(_worker, args=(world, _free_port(), n_total, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    o = oracle.Oracle(oracle.load_scene("ant"))
    qp = o.reset(n_total, 3, 0.1, 0.1)
    acts = synth.actions(4, 3, n_total, o.act_dim)
    for t in range(3):
        qp, _ = o.step(qp, acts[t])
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert float(d["steps"]) == n_total * 3          # SUM over ranks
        assert float(d["ms"]) == 10 + world - 1          # MAX over ranks
        assert float(d["blowups"]) == 0
        for k in ("pos", "rot", "vel", "ang"):
            assert np.array_equal(d[k], qp[k][int(d["lo"]):int(d["hi"])])


def _bench(args, env=None):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], capture_output=True, text=True,
                          cwd=root, env=e, timeout=300)


def test_bench_gpus2_starts_two_ranks_and_reduces_stats():
    """`python bench.py --gpus 2` (no launcher) starts 2 ranks itself (torch.distributed.run on
    127.0.0.1); they agree on WORLD_SIZE, build a 2-rank communicator and all-reduce the run
    statistics through the functions the B200 arm calls (dist.init_ranks, dist.barrier,
    dist.allreduce_stats) — here on gloo with synthetic per-rank numbers (--dist-selftest):
    SUM of env-steps 100 + 200, SUM of blow-ups 0 + 1, MAX of the times (10, 11 ms)."""
    import json
    r = _bench(["--gpus", "2", "--dist-selftest"])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["nranks"] == 2 and d["backend"] == "gloo"
    assert d["env_steps"] == 300.0 and d["blowups"] == 1.0 and d["ms_max"] == 11.0
    assert r.stderr.count("gloo communicator: nranks=2") == 2


def test_bench_rejects_a_world_size_mismatch():
    r = _bench(["--gpus", "2", "--dist-selftest"], env={"WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=3" in (r.stderr + r.stdout)


def test_torchrun_one_rank_builds_a_communicator():
    """Under the driver's launcher at N = 1 (torch.distributed.run, WORLD_SIZE = 1) the rank
    still builds its one-rank communicator and reduces through it (the launcher's path)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(root, "bench.py"),
                        "--gpus", "1", "--dist-selftest"], capture_output=True, text=True, env=e, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["n_gpus"] == 1 and d["nranks"] == 1 and d["backend"] == "gloo"
    assert d["env_steps"] == 100.0 and d["ms_max"] == 10.0
    assert "gloo communicator: nranks=1" in r.stderr
