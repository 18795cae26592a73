"""Pins of the oracle's directional derivative (oracle/diff.py, NEXT-4) against
closed forms: where the step is linear its Jacobian is the known update matrix."""
import numpy as np

import oracle
from oracle.diff import jvp_fd


def test_free_fall_jacobian_closed_form():
    """x' = x + S·h·v − g h² S(S+1)/2 (position-first symplectic Euler over S
    substeps): ∂x'/∂v = S·h = dt, ∂x'/∂x = 1, ∂v'/∂v = 1, ∂v'/∂x = 0."""
    txt = "dt: 0.02\nsubsteps: 4\ngravity { z: -9.8 }\nbodies { name: \"B\" mass: 2 inertia { x: 1 y: 1 z: 1 } }"
    o = oracle.Oracle(txt)
    qp = o.batch_default_qp(3)
    rng = np.random.default_rng(0)
    qp["vel"] = rng.normal(size=(3, 1, 3))
    dq = {k: np.zeros_like(v) for k, v in qp.items()}
    dq["vel"] = rng.normal(size=(3, 1, 3))
    dq["pos"] = rng.normal(size=(3, 1, 3))
    j, kink = jvp_fd(o, qp, None, dq, None)
    assert not kink.any()
    assert np.allclose(j["pos"], dq["pos"] + 0.02 * dq["vel"], atol=1e-8)
    assert np.allclose(j["vel"], dq["vel"], atol=1e-8)
    assert np.allclose(j["rot"], 0, atol=1e-8) and np.allclose(j["ang"], 0, atol=1e-8)


def test_axial_oscillator_jacobian_is_the_update_matrix_power():
    """A slider on a spring to a frozen parent (no rotation): the step is linear
    in (x, v) with matrix M^S, M = [[1, h], [−(k/m)h, 1 − (k/m)h² − (c/m)h]] on the
    axis (the oracle pin's recurrence), so J·v = M^S·v exactly."""
    k, c, m, h, S = 50.0, 0.5, 2.0, 0.005, 4
    txt = f"""dt: {h * S}
substeps: {S}
bodies {{ name: "P" frozen {{ all: true }} }}
bodies {{ name: "C" mass: {m} inertia {{ x: 1 y: 1 z: 1 }} frozen {{ rotation {{ x: 1 y: 1 z: 1 }} }} }}
joints {{ name: "J" parent: "P" child: "C" stiffness: {k} spring_damping: {c} angular_stiffness: 0
  limit_stiffness: 0 angle_limit {{ min: -180 max: 180 }} }}"""
    o = oracle.Oracle(txt)
    qp = o.batch_default_qp(1)
    qp["pos"][0, 1] = [0.1, -0.2, 0.05]
    qp["vel"][0, 1] = [0.3, 0.1, -0.4]
    M = np.array([[1.0, h], [-(k / m) * h, 1 - (k / m) * h * h - (c / m) * h]])
    MS = np.linalg.matrix_power(M, S)
    rng = np.random.default_rng(1)
    dq = {kk: np.zeros_like(v) for kk, v in qp.items()}
    dq["pos"][0, 1] = rng.normal(size=3)
    dq["vel"][0, 1] = rng.normal(size=3)
    j, kink = jvp_fd(o, qp, None, dq, None)
    assert not kink.any()
    for ax in range(3):
        want = MS @ np.array([dq["pos"][0, 1, ax], dq["vel"][0, 1, ax]])
        assert abs(j["pos"][0, 1, ax] - want[0]) < 1e-7
        assert abs(j["vel"][0, 1, ax] - want[1]) < 1e-7


def test_kink_detection_at_contact_activation():
    """The ball drop step at which contact begins is a kink along a height
    tangent (the ± evaluations differ in contact activity); a mid-air step is not."""
    o = oracle.Oracle(oracle.load_scene("ball"))
    qp = o.batch_default_qp(2)
    qp["pos"][0, 1, 2] = 0.5 + 1e-7   # touches the plane after this step's S2 for z − εdz
    qp["pos"][1, 1, 2] = 3.0
    qp["vel"][:, 1, 2] = 0.0
    dq = {k: np.zeros_like(v) for k, v in qp.items()}
    dq["pos"][:, 1, 2] = 1.0
    _, kink = jvp_fd(o, qp, None, dq, None, eps=1e-6)
    assert kink[0] and not kink[1]


def test_vjp_is_the_transposed_jvp():
    """⟨g, J·v⟩ = ⟨Jᵀ·g, v⟩ for random g, v (the adjoint identity), on a jointed
    scene with actions, and Jᵀg on the linear oscillator equals (M^S)ᵀ g."""
    from oracle.diff import jacobian_fd, vjp_fd
    o = oracle.Oracle(oracle.load_scene("chain2"))
    qp = o.reset(3, 1, 0.2, 0.2)
    rng = np.random.default_rng(2)
    a = rng.uniform(-1, 1, size=(3, o.act_dim))
    g = {k: rng.normal(size=v.shape) for k, v in qp.items()}
    v = {k: rng.normal(size=vv.shape) for k, vv in qp.items()}
    dv_a = rng.normal(size=(3, o.act_dim))
    jv, _ = jvp_fd(o, qp, a, v, dv_a)
    gin, ga, kink = vjp_fd(o, qp, a, g)
    assert not kink.any()
    lhs = sum((g[k] * jv[k]).reshape(3, -1).sum(1) for k in g)
    rhs = sum((gin[k] * v[k]).reshape(3, -1).sum(1) for k in g) + (ga * dv_a).sum(1)
    assert np.allclose(lhs, rhs, rtol=1e-6, atol=1e-6)
    J, _ = jacobian_fd(o, qp, a)
    assert J.shape == (3, 13 * o.n_bodies, 13 * o.n_bodies + o.act_dim)
