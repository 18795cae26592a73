"""GPU parity of the NEXT-4 forward-mode derivative (brax_step_jvp) against the
oracle's central differences (oracle/diff.py), away from the step's kinks."""
import numpy as np
import pytest

import oracle
import synth
from oracle.diff import jvp_fd

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
import paper_2106_13281_b200 as bx  # noqa: E402

FIELDS = ("pos", "rot", "vel", "ang")
# fp32 tangent arithmetic through S substeps vs an fp64 central difference, relative
# to the tangent's scale: measured ≤ 2.4e-5 over nine scenes, 8× margin
TOL_REL = 2e-4


def dev(q):
    return {k: torch.from_numpy(np.ascontiguousarray(q[k], dtype=np.float32)).cuda() for k in FIELDS}


def host(q):
    return {k: q[k].cpu().numpy().astype(np.float64) for k in FIELDS}


def states(o, n, seed, T0):
    qp = o.reset(n, seed, 0.1, 0.1)
    if T0:
        acts = synth.actions(seed + 1, T0, n, o.act_dim)
        for t in range(T0):
            qp, _ = o.step(qp, acts[t], threads=8)
    return synth.to_f32(qp)


def tangents(o, n, seed):
    rng = np.random.default_rng(seed)
    B = o.n_bodies
    dq = {"pos": rng.normal(size=(n, B, 3)), "rot": rng.normal(size=(n, B, 4)) * 0.1,
          "vel": rng.normal(size=(n, B, 3)), "ang": rng.normal(size=(n, B, 3))}
    for k in dq:  # static bodies never move: a tangent on them is meaningless
        for b, body in enumerate(o.sys.bodies):
            if body.is_static:
                dq[k][:, b] = 0
    dq = {k: v.astype(np.float32).astype(np.float64) for k, v in dq.items()}
    da = rng.normal(size=(n, o.act_dim)).astype(np.float32).astype(np.float64) if o.act_dim else None
    return dq, da


@pytest.mark.parametrize("name", ["pendulum", "chain2", "ball", "ant", "humanoid", "halfcheetah", "grasp", "fetch",
                                  "coverage"])
def test_jvp_matches_central_differences(name):
    text = oracle.load_scene(name)
    o, s = oracle.Oracle(text), bx.System(text)
    n = 200
    qp = states(o, n, seed=3, T0=5)
    act = synth.actions(4, 1, n, o.act_dim)[0] if o.act_dim else None
    dq, da = tangents(o, n, seed=5)
    ref, kink = jvp_fd(o, qp, act, dq, da, threads=8)
    keep = ~kink
    assert keep.mean() > 0.7, (~keep).sum()
    a_t = torch.from_numpy(act).cuda() if o.act_dim else None
    out, dout = s.step_jvp(dev(qp), a_t, dev(dq), torch.from_numpy(da.astype(np.float32)).cuda() if o.act_dim else None)
    # the primal is brax_step's output bit for bit
    plain = s.alloc_qp(n)
    s.step(dev(qp), a_t, plain)
    for k in FIELDS:
        assert torch.equal(out[k], plain[k]), k
    got = host(dout)
    for k in FIELDS:
        err = np.abs(got[k] - ref[k]).reshape(n, -1).max(1)
        scale = 1.0 + np.abs(ref[k]).reshape(n, -1).max(1)
        assert np.all(err[keep] <= TOL_REL * scale[keep]), (k, float((err / scale)[keep].max()))


def test_jacobian_columns_and_linear_case():
    """step_jacobian assembles unit-tangent JVPs; on the linear axial oscillator it
    equals the update matrix power M^S on each axis."""
    k, c, m, h, S = 50.0, 0.5, 2.0, 0.005, 4
    txt = f"""dt: {h * S}
substeps: {S}
bodies {{ name: "P" frozen {{ all: true }} }}
bodies {{ name: "C" mass: {m} inertia {{ x: 1 y: 1 z: 1 }} frozen {{ rotation {{ x: 1 y: 1 z: 1 }} }} }}
joints {{ name: "J" parent: "P" child: "C" stiffness: {k} spring_damping: {c} angular_stiffness: 0
  limit_stiffness: 0 angle_limit {{ min: -180 max: 180 }} }}"""
    o, s = oracle.Oracle(txt), bx.System(txt)
    qp = o.batch_default_qp(3)
    qp["pos"][:, 1] = [[0.1, -0.2, 0.05]] * 3
    jac = s.step_jacobian(dev(qp), None).cpu().numpy()
    M = np.array([[1.0, h], [-(k / m) * h, 1 - (k / m) * h * h - (c / m) * h]])
    MS = np.linalg.matrix_power(M, S)
    B = 2
    pos0, vel0 = 0, 7 * B        # column / row offsets of pos and vel blocks (pos 3B, rot 4B, vel 3B, ang 3B)
    for ax in range(3):
        ip, iv = pos0 + 3 + ax, vel0 + 3 + ax   # body 1
        assert np.allclose(jac[:, ip, ip], MS[0, 0], rtol=1e-5)
        assert np.allclose(jac[:, ip, iv], MS[0, 1], rtol=1e-5)
        assert np.allclose(jac[:, iv, ip], MS[1, 0], rtol=1e-5)
        assert np.allclose(jac[:, iv, iv], MS[1, 1], rtol=1e-5)


@pytest.mark.parametrize("name", ["pendulum", "chain2", "ant"])
def test_vjp_matches_transposed_central_differences(name):
    """brax_step_vjp (Jᵀ·g from the JVP columns) vs the oracle's Jᵀ·g with J by
    central differences; and the adjoint identity ⟨g, J·v⟩ = ⟨Jᵀg, v⟩ on the GPU."""
    from oracle.diff import vjp_fd
    text = oracle.load_scene(name)
    o, s = oracle.Oracle(text), bx.System(text)
    n = 48
    qp = states(o, n, seed=7, T0=3)
    act = synth.actions(8, 1, n, o.act_dim)[0] if o.act_dim else None
    rng = np.random.default_rng(9)
    g = {k: rng.normal(size=v.shape).astype(np.float32).astype(np.float64) for k, v in qp.items()}
    gin_ref, ga_ref, kink = vjp_fd(o, qp, act, g, threads=8)
    keep = ~kink
    assert keep.mean() > 0.7
    a_t = torch.from_numpy(act).cuda() if o.act_dim else None
    gin, ga = s.step_vjp(dev(qp), a_t, dev(g))
    got = host(gin)
    for k in FIELDS:
        err = np.abs(got[k] - gin_ref[k]).reshape(n, -1).max(1)
        scale = 1.0 + np.abs(gin_ref[k]).reshape(n, -1).max(1)
        assert np.all(err[keep] <= TOL_REL * scale[keep]), (k, float((err / scale)[keep].max()))
    if o.act_dim:
        err = np.abs(ga.cpu().numpy() - ga_ref).max(1)
        assert np.all(err[keep] <= TOL_REL * (1 + np.abs(ga_ref).max(1))[keep])
    # adjoint identity against the GPU's own JVP
    dq, da = tangents(o, n, seed=10)
    _, jv = s.step_jvp(dev(qp), a_t, dev(dq), torch.from_numpy(da.astype(np.float32)).cuda() if o.act_dim else None)
    jv = host(jv)
    lhs = sum((g[k] * jv[k]).reshape(n, -1).sum(1) for k in FIELDS)
    rhs = sum((got[k] * dq[k]).reshape(n, -1).sum(1) for k in FIELDS)
    if o.act_dim:
        rhs = rhs + (ga.cpu().numpy() * da).sum(1)
    assert np.allclose(lhs, rhs, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("name", ["coverage", "humanoid", "grasp"])
def test_fused_vjp_matches_the_column_vjp(name):
    """The one-launch reverse kernel (vjp.cu) and the JVP-column assembly (diff.cu)
    compute the same Jᵀ·g (two independent routes through the same derivative)."""
    import os
    text = oracle.load_scene(name)
    o, s = oracle.Oracle(text), bx.System(text)
    n = 70
    qp = states(o, n, seed=11, T0=4)
    act = synth.actions(12, 1, n, o.act_dim)[0]
    rng = np.random.default_rng(13)
    g = {k: rng.normal(size=v.shape).astype(np.float32) for k, v in qp.items()}
    a_t = torch.from_numpy(act).cuda()
    fused, fa = s.step_vjp(dev(qp), a_t, dev(g))
    os.environ["BRAX_VJP_COLUMNS"] = "1"
    try:
        cols, ca = s.step_vjp(dev(qp), a_t, dev(g))
    finally:
        os.environ.pop("BRAX_VJP_COLUMNS")
    for k in FIELDS:
        x, y = fused[k].cpu().numpy(), cols[k].cpu().numpy()
        scale = 1.0 + np.abs(y).reshape(n, -1).max(1)
        err = np.abs(x - y).reshape(n, -1).max(1)
        assert np.all(err <= 1e-4 * scale), (k, float((err / scale).max()))
    x, y = fa.cpu().numpy(), ca.cpu().numpy()
    assert np.all(np.abs(x - y).max(1) <= 1e-4 * (1 + np.abs(y).max(1)))


@pytest.mark.parametrize("name,T", [("pendulum", 20), ("chain2", 10), ("ant", 3)])
def test_trajectory_gradient_matches_oracle_rollout_differences(name, T):
    """APG-style gradient through a short trajectory: the loss
    L = Σ (final x of body 1) over envs; ⟨∇_a L, d⟩ from rollout_vjp equals the
    oracle rollout's central difference along random action directions d."""
    text = oracle.load_scene(name)
    o, s = oracle.Oracle(text), bx.System(text)
    n = 16
    qp = states(o, n, seed=21, T0=2)
    acts = synth.actions(22, T, n, o.act_dim)
    g_final = {k: torch.zeros(v.shape, device="cuda") for k, v in qp.items()}
    g_final["pos"][:, 1, 0] = 1.0
    _, g_a = s.rollout_vjp(dev(qp), torch.from_numpy(acts).cuda(), g_final)
    g_a = g_a.cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(23)
    d = rng.normal(size=acts.shape)

    def loss(a):
        q = {k: np.asarray(v, dtype=np.float64) for k, v in qp.items()}
        for t in range(T):
            q, _ = o.step(q, a[t], threads=8)
        return q["pos"][:, 1, 0]

    eps = 1e-5
    fd = (loss(acts + eps * d) - loss(acts - eps * d)) / (2 * eps)
    got = (g_a * d).sum(axis=(0, 2))
    assert np.allclose(got, fd, rtol=2e-3, atol=2e-4 * (1 + np.abs(fd).max())), np.abs(got - fd).max()


@pytest.mark.parametrize("name", ["coverage", "ant"])
def test_hand_joint_adjoint_matches_local_derivatives(name):
    """The hand-derived joint adjoint (vjp.cu joint_adj) and the local value+tangent
    evaluations of the same joint code (BRAX_VJP_LOCAL_AD=1) give the same Jᵀ·g."""
    import os
    text = oracle.load_scene(name)
    o, s = oracle.Oracle(text), bx.System(text)
    n = 64
    qp = states(o, n, seed=31, T0=3)
    act = synth.actions(32, 1, n, o.act_dim)[0]
    rng = np.random.default_rng(33)
    g = {k: rng.normal(size=v.shape).astype(np.float32) for k, v in qp.items()}
    a_t = torch.from_numpy(act).cuda()
    hand, ha = s.step_vjp(dev(qp), a_t, dev(g))
    os.environ["BRAX_VJP_LOCAL_AD"] = "1"
    try:
        loc, la = s.step_vjp(dev(qp), a_t, dev(g))
    finally:
        os.environ.pop("BRAX_VJP_LOCAL_AD")
    for k in FIELDS:
        x, y = hand[k].cpu().numpy(), loc[k].cpu().numpy()
        scale = 1.0 + np.abs(y).reshape(n, -1).max(1)
        assert np.all(np.abs(x - y).reshape(n, -1).max(1) <= 1e-4 * scale), k
    x, y = ha.cpu().numpy(), la.cpu().numpy()
    assert np.all(np.abs(x - y).max(1) <= 1e-4 * (1 + np.abs(y).max(1)))
