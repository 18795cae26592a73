"""GPU parity of the NEXT-1 env epilogue (brax_env_step / brax_env_reset /
brax_env_observe through the C ABI) against the oracle's env (oracle/env.py) on
identical seeded fp32 inputs.  Tolerances: the step's 1e-4 on the QP (BASELINE
north_star); observations share it; reward = Δx·f/dt + ... inherits
TOL_STEP·|f|/dt; done, steps and episode bit-exact outside a 1e-4 band around the
height thresholds and outside the R23 ambiguity band."""
import os

import numpy as np
import pytest

import oracle
import synth
from oracle.env import Env

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
import paper_2106_13281_b200 as bx  # noqa: E402

TOL = 1e-4
FIELDS = ("pos", "rot", "vel", "ang")
ENV_SCENES = ["ant", "humanoid", "halfcheetah", "grasp", "fetch"]
_cache = {}


def scene(name):
    if name not in _cache:
        text = oracle.load_scene(name)
        _cache[name] = (Env(oracle.Oracle(text)), bx.System(text))
    return _cache[name]


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dtype).cuda()


def start_states(e, n, seed):
    """Reset states advanced 0-12 steps by the oracle (varied contacts), and step
    counters that put some envs on their truncation step."""
    rng = np.random.default_rng(seed)
    qp = e.o.reset(n, seed, 0.1, 0.1)
    acts = synth.actions(seed + 1, 12, n, e.sys.act_dim)
    T = rng.integers(0, 13, size=n)
    for t in range(12):
        nxt, _ = e.o.step(qp, acts[t], threads=8)
        m = T > t
        for k in qp:
            qp[k][m] = nxt[k][m]
    qp = synth.to_f32(qp)
    L = e.task.episode_length
    steps = np.where(rng.random(n) < 0.2, L - 1, rng.integers(0, L - 1, size=n)).astype(np.int32)
    episode = rng.integers(0, 5, size=n).astype(np.uint32)
    return qp, steps, episode


def near_threshold(e, z, d1=None):
    """Envs whose fp32 decision (height limits; goal tasks: the marker radius, R36) lies
    within the step tolerance of its threshold."""
    out = np.zeros_like(z, dtype=bool)
    if e.task.healthy_z is not None:
        lo, hi = e.task.healthy_z
        out |= (np.abs(z - lo) < TOL) | (np.abs(z - hi) < TOL)
    if d1 is not None:
        out |= np.abs(d1 - e.task.goal.radius) < 2 * TOL
    return out


def near_marker(e, qp, seed, frac=0.4):
    """Goal tasks: put the marker within about the radius of the object in a fraction
    of the envs, so that hits (bonus + new marker) occur in the step."""
    g = e.task.goal
    if g is None:
        return qp
    rng = np.random.default_rng(seed)
    n = qp["pos"].shape[0]
    m = rng.random(n) < frac
    d = rng.normal(size=(n, 3))
    d *= (g.radius * rng.uniform(0.3, 1.3, size=(n, 1))) / np.linalg.norm(d, axis=1, keepdims=True)
    qp["pos"][m, g.target] = (qp["pos"][m, g.obj] + d[m]).astype(qp["pos"].dtype)
    return qp


@pytest.mark.parametrize("name", ENV_SCENES)
def test_env_reset_and_observe(name):
    e, s = scene(name)
    n = 333
    st = s.env_state(n)
    obs = s.env_reset(st, seed=17, env_offset=1000).cpu().numpy()
    qp, steps, ep, obs_ref = e.reset(n, seed=17, env_offset=1000)
    for k in FIELDS:
        assert np.max(np.abs(st["qp"][k].cpu().numpy() - qp[k])) < 1e-6, k
    assert not st["steps"].any() and not st["episode"].any()
    assert obs.shape == (n, e.obs_dim)
    assert np.max(np.abs(obs - obs_ref)) < TOL
    # observe leaves the QP alone and repeats the reset's observation bitwise
    before = {k: v.clone() for k, v in st["qp"].items()}
    again = s.env_observe(st["qp"]).cpu().numpy()
    assert np.array_equal(again, obs)
    for k in FIELDS:
        assert torch.equal(before[k], st["qp"][k])


@pytest.mark.parametrize("name", ENV_SCENES)
def test_env_step_matches_oracle(name):
    e, s = scene(name)
    n = 1000
    qp, steps, ep = start_states(e, n, seed=31)
    qp = near_marker(e, qp, seed=33)
    act = synth.actions(32, 1, n, e.sys.act_dim)[0]
    ref = e.step(qp, steps, ep, act, seed=9, env_offset=50, threads=8)
    st = {"qp": {k: dev(qp[k]) for k in FIELDS}, "steps": dev(steps, torch.int32),
          "episode": dev(ep.view(np.int32), torch.int32)}
    out = s.env_step(st, dev(act), seed=9, env_offset=50)
    keep = ~ref["ambiguous"] & ~near_threshold(e, ref["x1_z"], ref["d1"])
    assert keep.mean() > 0.9
    done = out["done"][0].cpu().numpy().astype(bool)
    assert np.array_equal(done[keep], ref["done"][keep])
    assert ref["done"].sum() >= 0.1 * n  # the truncation envs at least
    assert np.array_equal(st["steps"].cpu().numpy()[keep], ref["steps"][keep])
    assert np.array_equal(st["episode"].cpu().numpy().view(np.uint32)[keep], ref["episode"][keep])
    if e.task.goal is None:
        tol_r = 2 * TOL * np.linalg.norm(e.task.forward, 1) / e.sys.dt + 1e-5
    else:  # |Δd1| ≤ |Δx'| plus fp32 rounding of the distances (R36)
        hits = ref["d1"] < e.task.goal.radius
        assert hits[keep].sum() >= 0.1 * n, hits.sum()
        tol_r = (2 * TOL + 4e-7 * (1 + np.max(ref["d1"]))) / e.sys.dt + 1e-5
    r = out["reward"][0].cpu().numpy()
    assert np.max(np.abs(r[keep] - ref["reward"][keep])) < tol_r
    for k in FIELDS:
        got = st["qp"][k].cpu().numpy()
        assert np.max(np.abs(got[keep] - ref["qp"][k][keep])) < TOL, k
    obs = out["obs"][0].cpu().numpy()
    assert np.max(np.abs(obs[keep] - ref["obs"][keep])) < TOL


@pytest.mark.parametrize("name", ["ant", "grasp"])
def test_env_rollout_equals_single_steps_and_plans_agree(name):
    """T steps in one launch give the same bits as T single-step launches, and
    every launch plan gives the same bits (auto-resets and marker hits included)."""
    e, s = scene(name)
    n = 500
    qp, steps, ep = start_states(e, n, seed=41)
    qp = near_marker(e, qp, seed=43)
    T = 6
    acts = dev(synth.actions(42, T, n, e.sys.act_dim))

    def fresh():
        return {"qp": {k: dev(qp[k]) for k in FIELDS}, "steps": dev(steps, torch.int32),
                "episode": dev(ep.view(np.int32), torch.int32)}

    a = fresh()
    big = s.env_step(a, acts, seed=3)
    b = fresh()
    small = [s.env_step(b, acts[t], seed=3) for t in range(T)]
    for key in ("obs", "reward", "done"):
        assert torch.equal(big[key], torch.cat([o[key] for o in small])), key
    for k in FIELDS:
        assert torch.equal(a["qp"][k], b["qp"][k]), k
    assert torch.equal(a["steps"], b["steps"]) and torch.equal(a["episode"], b["episode"])
    assert big["done"].sum() > 0
    try:
        for plan, fixed in (("2,1", "0"), ("4,1", "0"), ("1,2", "0"), ("2,2", "0"), ("4,2", "0"), ("1,2", "1"),
                            ("2,2", "1"), ("4,2", "1")):
            os.environ["BRAX_PLAN"] = plan
            os.environ["BRAX_FIXED_GATHER"] = fixed
            c = fresh()
            other = s.env_step(c, acts, seed=3)
            for key in ("obs", "reward", "done"):
                assert torch.equal(other[key], big[key]), (plan, key)
            for k in FIELDS:
                assert torch.equal(c["qp"][k], a["qp"][k]), (plan, k)
    finally:
        os.environ.pop("BRAX_PLAN", None)
        os.environ.pop("BRAX_FIXED_GATHER", None)


def test_env_errors():
    _, s = scene("ant")
    plain = bx.System(oracle.load_scene("ball"))
    st = plain.env_state(4)
    with pytest.raises(bx.BraxError, match="no task"):
        plain.env_reset(st)
    st = s.env_state(4)
    s.env_reset(st)
    with pytest.raises(bx.BraxError):
        bx.brax_env_step(s.handle, st["qp"], None, 1, st["qp"], 4, None, None, None, None, None)


@pytest.mark.parametrize("name", ENV_SCENES)
def test_lean_kernel_env_and_random_actions_bit_identical(name):
    """The lean kernel's env-epilogue and on-device-action paths give brax_step_kernel's bits
    (same device code in the same order) for every plan it applies to."""
    import os
    o = oracle.Oracle(oracle.load_scene(name))
    s = bx.System(oracle.load_scene(name))
    n, T = 300, 3
    acts = torch.from_numpy(synth.actions(31, T, n, o.act_dim)).cuda()
    q0 = o.reset(n, 32, 0.1, 0.1)

    def run(plan, lean):
        os.environ.update({"BRAX_PLAN": plan, "BRAX_LEAN": lean, "BRAX_FIXED_GATHER": "1"})
        try:
            st = s.env_state(n)
            s.env_reset(st, seed=4)
            out = s.env_step(st, acts, seed=4)
            qr = {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda() for k, v in q0.items()}
            s.rollout_random(qr, T, seed=9, env_offset=3, step0=2)
            torch.cuda.synchronize()
            return out, st, qr
        finally:
            for k in ("BRAX_PLAN", "BRAX_LEAN", "BRAX_FIXED_GATHER"):
                os.environ.pop(k, None)
    for plan in ("2,2", "4,2", "2,1", "4,1"):
        ref, st_ref, qr_ref = run(plan, "0")
        got, st_got, qr_got = run(plan, "1")
        for key in ("obs", "reward", "done"):
            assert torch.equal(got[key], ref[key]), (plan, key)
        for k in ("pos", "rot", "vel", "ang"):
            assert torch.equal(st_got["qp"][k], st_ref["qp"][k]), (plan, k)
            assert torch.equal(qr_got[k], qr_ref[k]), (plan, k)
        assert torch.equal(st_got["steps"], st_ref["steps"]) and torch.equal(st_got["episode"], st_ref["episode"])
