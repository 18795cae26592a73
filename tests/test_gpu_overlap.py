"""Launch overlap of the lean step kernel (DESIGN.md §5 "Launch overlap"): consecutive
launches on a stream skip the grid-wide dependent-launch wait and order themselves per
env granule through device counters.  A missed dependency would read a stale QP, so
every sequence here — in-place chains, rotating buffer sets, plan / kernel / batch-size
changes between launches, sub-views of one buffer, CUDA graphs, two streams — must give
the bits of the same launches run one at a time with a device synchronisation between
them (no overlap possible).  The step's arithmetic does not depend on the overlap."""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
import paper_2106_13281_b200 as bx  # noqa: E402

FIELDS = ("pos", "rot", "vel", "ang")


def start(o, n, seed):
    return {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda()
            for k, v in o.reset(n, seed, 0.1, 0.1).items()}


def clone(q):
    return {k: v.clone() for k, v in q.items()}


def view(q, lo, hi):
    return {k: v[lo:hi] for k, v in q.items()}


def run(s, ops, sync):
    """ops: callables (s) -> None launching one step each; sync: device sync after each."""
    for op in ops:
        op(s)
        if sync:
            torch.cuda.synchronize()
    torch.cuda.synchronize()


def with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("n", [8192, 1000])
def test_in_place_chain_matches_serialised_launches(n):
    o = oracle.Oracle(oracle.load_scene("ant"))
    s = bx.System(oracle.load_scene("ant"))
    q0 = start(o, n, 1)
    acts = torch.from_numpy(synth.actions(2, 60, n, o.act_dim)).cuda()
    s.tune(q0, acts[0])
    got, ref = clone(q0), clone(q0)
    run(s, [lambda s, t=t: s.step(got, acts[t], got) for t in range(60)], sync=False)
    run(s, [lambda s, t=t: s.step(ref, acts[t], ref) for t in range(60)], sync=True)
    for k in FIELDS:
        assert torch.equal(got[k], ref[k]), k


def test_mixed_plans_kernels_views_and_rotation():
    """Plan changes (granules shared by blocks of different sizes), generic launches in
    between (contact_dp forces brax_step_kernel), sub-views of the batch (partial
    overlaps: full wait) and a second buffer set, in one stream."""
    o = oracle.Oracle(oracle.load_scene("ant"))
    s = bx.System(oracle.load_scene("ant"))
    n = 4096
    A0, B0 = start(o, n, 3), start(o, n, 4)
    acts = torch.from_numpy(synth.actions(5, 40, n, o.act_dim)).cuda()
    cdp = torch.empty((n, s.n_bodies, 6), device="cuda")
    plans = [("4,2", "1"), ("2,2", "1"), ("4,1", "1"), ("4,2", "0"), ("2,1", "1"), ("4,2", "1")]

    def ops(A, Bq):
        out = []
        for t in range(40):
            plan, lean = plans[t % len(plans)]
            env = {"BRAX_PLAN": plan, "BRAX_LEAN": lean, "BRAX_FIXED_GATHER": "1"}
            if t % 7 == 3:
                out.append(lambda s, t=t, env=env: with_env(env, lambda: s.step(A, acts[t], A, contact_dp=cdp)))
            elif t % 5 == 2:
                out.append(lambda s, t=t, env=env: with_env(env, lambda: s.step(view(A, 0, 1000), acts[t][:1000],
                                                                                  view(A, 0, 1000))))
            elif t % 5 == 4:
                out.append(lambda s, t=t, env=env: with_env(env, lambda: s.step(view(A, 992, n), acts[t][992:],
                                                                                  view(A, 992, n))))
            else:
                out.append(lambda s, t=t, env=env: with_env(env, lambda: s.step(A, acts[t], A)))
            out.append(lambda s, t=t, env=env: with_env(env, lambda: s.step(Bq, acts[t], Bq)))
        return out
    A1, B1 = clone(A0), clone(B0)
    A2, B2 = clone(A0), clone(B0)
    run(s, ops(A1, B1), sync=False)
    run(s, ops(A2, B2), sync=True)
    for k in FIELDS:
        assert torch.equal(A1[k], A2[k]), k
        assert torch.equal(B1[k], B2[k]), k


def test_graph_of_chained_and_rotating_launches():
    """A CUDA graph (the bench's launch form) of in-place and ping-pong launches, replayed
    three times, against the same launches serialised."""
    o = oracle.Oracle(oracle.load_scene("halfcheetah"))
    s = bx.System(oracle.load_scene("halfcheetah"))
    n = 4096
    q0 = start(o, n, 7)
    acts = torch.from_numpy(synth.actions(8, 24, n, o.act_dim)).cuda()
    s.tune(q0, acts[0])
    X, Y = clone(q0), s.alloc_qp(n)

    def seq():
        for t in range(24):
            if t % 3 == 2:
                s.step(X, acts[t], Y)  # ping-pong: the next launch reads what this one wrote
                s.step(Y, acts[t], X)
            else:
                s.step(X, acts[t], X)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        seq()
    torch.cuda.synchronize()
    X.update(clone(q0))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        seq()
    for k in FIELDS:
        X[k].copy_(q0[k])
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    R, RY = clone(q0), s.alloc_qp(n)
    for _ in range(3):
        for t in range(24):
            if t % 3 == 2:
                s.step(R, acts[t], RY)
                torch.cuda.synchronize()
                s.step(RY, acts[t], R)
            else:
                s.step(R, acts[t], R)
            torch.cuda.synchronize()
    for k in FIELDS:
        assert torch.equal(X[k], R[k]), k


def test_two_streams_share_a_system():
    """Two streams step disjoint batches of one system concurrently (their launches meet on
    the same granule counters): no deadlock, and each batch gets its serialised bits."""
    o = oracle.Oracle(oracle.load_scene("ant"))
    s = bx.System(oracle.load_scene("ant"))
    n = 2048
    P0, Q0 = start(o, n, 11), start(o, n, 12)
    acts = torch.from_numpy(synth.actions(13, 30, n, o.act_dim)).cuda()
    P, Q = clone(P0), clone(Q0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for t in range(30):
        with torch.cuda.stream(s1):
            s.step(P, acts[t], P, stream=s1)
        with torch.cuda.stream(s2):
            s.step(Q, acts[t], Q, stream=s2)
    torch.cuda.synchronize()
    RP, RQ = clone(P0), clone(Q0)
    run(s, [lambda s, t=t: s.step(RP, acts[t], RP) for t in range(30)], sync=True)
    run(s, [lambda s, t=t: s.step(RQ, acts[t], RQ) for t in range(30)], sync=True)
    for k in FIELDS:
        assert torch.equal(P[k], RP[k]) and torch.equal(Q[k], RQ[k]), k


@pytest.mark.parametrize("scene,plan,lean", [("ant", None, None), ("ant", "4,2", "0"), ("ant", "1,2", "0"),
                                             ("ant", "2,1", "1"), ("grasp", None, None)])
def test_env_chain_matches_serialised_launches(scene, plan, lean):
    """Env launches (reward / done / auto-reset / observations; grasp: goal markers) overlapped,
    lean and generic kernels, against the same launches serialised."""
    o = oracle.Oracle(oracle.load_scene(scene))
    s = bx.System(oracle.load_scene(scene))
    n = 2000
    acts = torch.from_numpy(synth.actions(21, 40, n, o.act_dim)).cuda()
    env = {} if plan is None else {"BRAX_PLAN": plan, "BRAX_LEAN": lean, "BRAX_FIXED_GATHER": "1"}

    def go(sync):
        return with_env(env, lambda: go_(sync))

    def go_(sync):
        st = s.env_state(n)
        s.env_reset(st, seed=5)
        outs = []
        for t in range(40):
            outs.append(s.env_step(st, acts[t], seed=5))
            if sync:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        return st, outs
    a, oa = go(False)
    b, ob = go(True)
    for k in FIELDS:
        assert torch.equal(a["qp"][k], b["qp"][k]), k
    for x, y in zip(oa, ob):
        for key in ("obs", "reward", "done"):
            assert torch.equal(x[key], y[key]), key


def test_eager_launches_right_after_a_graph_replay():
    """A replayed graph of in-place launches, then eager launches on the same buffers and
    stream with no synchronisation: the eager launches' record predates the capture (a
    capture tracks its own order), and the graph launch serialises with them."""
    o = oracle.Oracle(oracle.load_scene("ant"))
    s = bx.System(oracle.load_scene("ant"))
    n = 8192
    q0 = start(o, n, 31)
    acts = torch.from_numpy(synth.actions(32, 16, n, o.act_dim)).cuda()
    X = clone(q0)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        s.step(X, acts[0], X)  # the stream's eager record: an in-place launch on X
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for t in range(1, 9):
            s.step(X, acts[t], X)
    for k in FIELDS:
        X[k].copy_(q0[k])
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        s.step(X, acts[0], X)
        g.replay()
        for t in range(9, 16):
            s.step(X, acts[t], X)
    torch.cuda.synchronize()
    R = clone(q0)
    run(s, [lambda s, t=t: s.step(R, acts[t], R) for t in range(16)], sync=True)
    for k in FIELDS:
        assert torch.equal(X[k], R[k]), k
