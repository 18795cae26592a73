"""Pins of the fp64 oracle against closed forms, invariants, textbook routines
and brute force.  None of these re-types the oracle's
formulas: each expected value comes from the mathematics of the discrete map
(derivations in DESIGN.md "Oracle pins") or from an independent library
(scipy) or from brute force.  CPU only.
"""
import math
import os

import numpy as np
import pytest

import oracle
from oracle.philox import philox4x32_10

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    vals = {}
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, *v = line.split()
            vals[k] = v
    return vals


CF = golden("closed_forms.txt")


def cf(key):
    return float(CF[key][0])


def single_body(gravity=-9.8, dt=0.01, substeps=1, extra=""):
    return f"""
dt: {dt}
substeps: {substeps}
gravity {{ z: {gravity} }}
bodies {{ name: "B" mass: 1 inertia {{ x: 1 y: 1 z: 1 }} }}
{extra}
"""


def qp1(o, **kw):
    q = o.batch_default_qp(1)
    for k, v in kw.items():
        q[k][0] = v
    return q


# ---------------------------------------------------------------- kinematics
def test_free_fall_closed_form():
    """x_z(N) = z0 − g h² N(N−1)/2, v_z(N) = −g N h, ΔE = ½ m g² h² N (position-first
    symplectic Euler, Alg. 1)."""
    o = oracle.Oracle(single_body())
    q = o.batch_default_qp(1)
    E0 = 0.0
    for _ in range(100):
        q, _ = o.step(q)
    z, vz = q["pos"][0, 0, 2], q["vel"][0, 0, 2]
    assert abs(z - cf("free_fall_z")) < 1e-12
    assert abs(vz - cf("free_fall_vz")) < 1e-12
    E = 0.5 * vz * vz + 9.8 * z
    assert abs((E - E0) - 0.5 * 9.8 ** 2 * 0.01 ** 2 * 100) < 1e-12
    assert abs((E - E0) - cf("free_fall_dE")) < 1e-12
    # continuous ballistics is within ½·g·t·h of the discrete map
    assert abs(z - (-0.5 * 9.8 * 1.0 ** 2)) <= 0.5 * 9.8 * 1.0 * 0.01 + 1e-12


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_spin_closed_form(axis):
    """q ← normalize(q + ½h(0,ω)⊗q) rotates by exactly 2·atan(ωh/2) per substep
    about a fixed axis (R3); 1000 substeps at ω = π, h = 1e-3."""
    o = oracle.Oracle(single_body(gravity=0, dt=1e-3))
    w = np.zeros(3)
    w[axis] = math.pi
    q = qp1(o, ang=[w])
    for _ in range(1000):
        q, _ = o.step(q)
    r = q["rot"][0, 0]
    theta = 2 * math.atan2(np.linalg.norm(r[1:]), r[0])
    assert abs(theta - 2 * 1000 * math.atan(math.pi * 1e-3 / 2)) < 1e-12
    assert abs(theta - cf("spin_theta")) < 1e-12
    assert abs(np.linalg.norm(r) - 1) < 1e-14
    assert abs(r[1 + axis] - math.sin(theta / 2)) < 1e-12


def test_frozen_masks_bitwise():
    """Frozen axes (App. A `frozen`; masks R21): a fully frozen body is
    bitwise unchanged; a planar body keeps pos.y and has zero v.y, ω.x, ω.z."""
    txt = """dt: 0.01 gravity { z: -9.8 }
bodies { name: "F" frozen { all: true } }
bodies { name: "P" frozen { position { y: 1 } rotation { x: 1 z: 1 } } }"""
    o = oracle.Oracle(txt)
    q = o.batch_default_qp(3)
    rng = np.random.default_rng(1)
    for k in q:
        q[k] = rng.normal(size=q[k].shape)
    q["rot"] /= np.linalg.norm(q["rot"], axis=-1, keepdims=True)
    q0 = {k: v.copy() for k, v in q.items()}
    for _ in range(10):
        q, _ = o.step(q)
    for k in q:
        assert np.array_equal(q[k][:, 0], q0[k][:, 0])
    assert np.array_equal(q["pos"][:, 1, 1], q0["pos"][:, 1, 1])
    assert np.all(q["vel"][:, 1, 1] == 0) and np.all(q["ang"][:, 1, [0, 2]] == 0)


# ---------------------------------------------------------------- joints
def axial_oscillator(c):
    return f"""dt: 0.01 substeps: 1
bodies {{ name: "P" frozen {{ all: true }} }}
bodies {{ name: "C" mass: 1 inertia {{ x: 1 y: 1 z: 1 }} }}
joints {{ name: "J" parent: "P" child: "C" stiffness: 10000 spring_damping: {c}
  angle_limit {{ min: -180 max: 180 }} }}"""


@pytest.mark.parametrize("c", [0.0, 5.0])
def test_axial_oscillator_matrix_power(c):
    """Linear spring-damper at the anchors (R5) + symplectic Euler: (x, v) follows
    M = [[1, h], [−(k/m)h, 1 − (k/m)h² − (c/m)h]] raised to the n-th power."""
    o = oracle.Oracle(axial_oscillator(c))
    k, m, h = 1e4, 1.0, 0.01
    M = np.array([[1, h], [-(k / m) * h, 1 - (k / m) * h * h - (c / m) * h]])
    q = qp1(o, pos=[[0, 0, 0], [0.1, 0, 0]], vel=[[0, 0, 0], [0.3, 0, 0]])
    s0 = np.array([0.1, 0.3])
    for n in range(1, 40):
        q, _ = o.step(q)
        sn = np.linalg.matrix_power(M, n) @ s0
        assert abs(q["pos"][0, 1, 0] - sn[0]) < 1e-12
        assert abs(q["vel"][0, 1, 0] - sn[1]) < 1e-12
    if c == 0:  # Ωh = π/3: period exactly 6 substeps
        assert np.allclose(np.linalg.matrix_power(M, 6), np.eye(2), atol=1e-12)


def test_hooke_force():
    """0.1 m × 10000 N/m → 1000 N on the child: Δv = F·h/m = 10 m/s."""
    o = oracle.Oracle(axial_oscillator(0.0))
    q = qp1(o, pos=[[0, 0, 0], [0, 0, 0.1]])
    q, _ = o.step(q)
    # the kinematic step leaves x unchanged (v = 0), so F = k·(−0.1) along z
    assert abs(q["vel"][0, 1, 2] - (-1000 * 0.01)) < 1e-12


def test_torsional_oscillator_recurrence():
    """Hinge with limits [0, 0] (R7, R8): θ_{n+1} = θ_n + 2·atan(ω_n h/2);
    ω_{n+1} = ω_n − (k_l/I)·θ_{n+1}·h."""
    txt = """dt: 0.01
bodies { name: "P" frozen { all: true } }
bodies { name: "C" mass: 1 inertia { x: 2 y: 2 z: 2 } }
joints { name: "J" parent: "P" child: "C" stiffness: 1000 limit_stiffness: 300
  angle_limit { min: 0 max: 0 } }"""
    o = oracle.Oracle(txt)
    q = qp1(o, ang=[[0, 0, 0], [0.7, 0, 0]])
    th, w = 0.0, 0.7
    for _ in range(300):
        q, _ = o.step(q)
        th = th + 2 * math.atan(w * 0.01 / 2)
        w = w - (300 / 2) * th * 0.01
        r = q["rot"][0, 1]
        assert abs(2 * math.atan2(r[1], r[0]) - th) < 1e-12
        assert abs(q["ang"][0, 1, 0] - w) < 1e-12


def test_alignment_torque_about_the_rotated_euler_axis():
    """R7 (as amended): the alignment spring of axis 1 acts about
    a1 = Rx(θ0)·ŷ.  A hinge at angle θ0 = 0.5 (free, inside its limits) with an
    alignment error α about that rotated axis therefore rotates about the fixed
    axis a1 only: α follows the scalar recurrence α_{n+1} = α_n + 2·atan(ω_n h/2),
    ω_{n+1} = ω_n − (k_a/I)·α_{n+1}·h, and θ0 stays 0.5."""
    txt = """dt: 0.01
bodies { name: "P" frozen { all: true } }
bodies { name: "C" mass: 1 inertia { x: 2 y: 2 z: 2 } }
joints { name: "J" parent: "P" child: "C" stiffness: 1000 angular_stiffness: 400
  angle_limit { min: -60 max: 60 } }"""
    o = oracle.Oracle(txt)
    th0, alpha = 0.5, 0.03
    a1 = np.array([0.0, math.cos(th0), math.sin(th0)])
    qx = np.array([math.cos(th0 / 2), math.sin(th0 / 2), 0, 0])
    qa = np.array([math.cos(alpha / 2), *(math.sin(alpha / 2) * a1)])  # rotation about a1 by α
    qc = oracle.system.qmul(qa, qx)                                    # = Rx(θ0)·Ry(α)
    q = qp1(o, rot=[[1, 0, 0, 0], qc])
    al, w = alpha, 0.0
    for _ in range(200):
        q, _ = o.step(q)
        al = al + 2 * math.atan(w * 0.01 / 2)
        w = w - (400 / 2) * al * 0.01
        r = q["rot"][0, 1]
        # relative rotation back to the hinge: conj(qx) = rotation about a1 by the current α
        rel = oracle.system.qmul(r, oracle.system.qconj(qx))
        assert abs(2 * math.atan2(np.dot(rel[1:], a1), rel[0]) - al) < 1e-10
        assert np.allclose(q["ang"][0, 1], w * a1, atol=1e-10)


@pytest.mark.parametrize("dof", [1, 2, 3])
def test_joint_torque_is_the_spring_potential_gradient(dof):
    """R7 (as amended): the angular-spring torque on the child is −∂V/∂φ, V = ½k_l Σ_{i<dof}
    (θ_i − clamp θ_i)² + ½k_a Σ_{i≥dof} θ_i², φ a world-frame rotation of the child — the
    conservative force PAPER.md:264's energy behaviour needs.  V is evaluated here by an
    independent numpy Euler extraction and differentiated by central differences; the
    oracle's torque is read from one substep of an iso-inertia child: Δω = h·τ/I."""
    import sys as _sys
    _sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    import astronaut
    lims = " ".join(["angle_limit { min: -10 max: 10 }", "angle_limit { min: -5 max: 5 }",
                     "angle_limit { min: -8 max: 12 }"][:dof])
    txt = f"""dt: 0.001
substeps: 1
bodies {{ name: "P" frozen {{ all: true }} }}
bodies {{ name: "C" mass: 1 inertia {{ x: 2 y: 2 z: 2 }} }}
joints {{ name: "J" parent: "P" child: "C" stiffness: 1000 angular_stiffness: 300
  limit_stiffness: 500 rotation {{ z: 30 x: 20 }} reference_rotation {{ y: 15 }} {lims} }}"""
    o = oracle.Oracle(txt)
    j = o.sys.joints[0]
    rng = np.random.default_rng(dof)
    for _ in range(5):
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        ang = rng.uniform(0.2, 0.8)
        qc = np.array([math.cos(ang / 2), *(math.sin(ang / 2) * ax)])
        qp0 = np.array([1.0, 0, 0, 0])

        def V(q):
            th = astronaut.joint_angles(qp0[None], q[None], j)[0]
            v = 0.0
            for i in range(3):
                if i < dof:
                    v += 0.5 * j.limit_stiffness * (th[i] - np.clip(th[i], *j.limits[i])) ** 2
                else:
                    v += 0.5 * j.angular_stiffness * th[i] ** 2
            return v
        eps = 1e-6
        grad = np.zeros(3)
        for k in range(3):
            d = np.zeros(3)
            d[k] = eps
            qplus = oracle.system.qmul(np.array([math.cos(eps / 2), *(math.sin(eps / 2) * d / eps)]), qc)
            qminus = oracle.system.qmul(np.array([math.cos(eps / 2), *(-math.sin(eps / 2) * d / eps)]), qc)
            grad[k] = (V(qplus) - V(qminus)) / (2 * eps)
        q = qp1(o, rot=[qp0, qc])
        q, _ = o.step(q)
        tau = q["ang"][0, 1] * 2.0 / 0.001
        assert np.linalg.norm(grad) > 1.0
        assert np.allclose(tau, -grad, rtol=1e-6, atol=1e-6 * np.linalg.norm(grad)), (tau, -grad)


def test_undamped_energy_drift_shrinks_with_h():
    """Fig. 5 energy protocol in fp64: the undamped, gravity- and
    contact-free humanoid kicked at 1 m/s keeps its energy to O(h), and the drift
    after 1 s shrinks as the substep halves."""
    import sys as _sys
    _sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    import astronaut
    drifts = []
    for S in (2, 4, 8):
        o = oracle.Oracle(astronaut.astronaut_text(S, 0.0))
        qp = o.batch_default_qp(8)
        kick = np.random.default_rng(0).normal(size=qp["vel"].shape)
        qp["vel"] = kick / np.linalg.norm(kick, axis=-1, keepdims=True)
        E0 = astronaut.invariants(o.sys, qp)[2]
        for _ in range(67):
            qp, _ = o.step(qp, np.zeros((8, o.act_dim)))
        drifts.append(np.abs(astronaut.invariants(o.sys, qp)[2] - E0).mean() / E0.mean())
    assert drifts[0] < 0.15 and drifts[1] < drifts[0] and drifts[2] < drifts[1], drifts


def test_angle_actuator_servo_recurrence():
    """ANGLE actuator (R12): τ = s·(clamp(a, lo, hi) − θ) about the free axis; with wide
    limits and no other torque: θ_{n+1} = θ_n + 2·atan(ω_n h/2), ω_{n+1} = ω_n +
    (s·(a − θ_{n+1}) + k_l·(clamp(θ_{n+1}, lo, hi) − θ_{n+1}))·h/I; the target a is
    clamped to the limits."""
    txt = """dt: 0.01
bodies { name: "P" frozen { all: true } }
bodies { name: "C" mass: 1 inertia { x: 0.5 y: 0.5 z: 0.5 } }
joints { name: "J" parent: "P" child: "C" stiffness: 1000 angle_limit { min: -90 max: 60 } }
actuators { name: "J" joint: "J" strength: 20 angle {} }"""
    o = oracle.Oracle(txt)
    for target in (0.4, 2.0):  # 2.0 rad is beyond the 60° limit: clamped to π/3
        q = o.batch_default_qp(1)
        th, w = 0.0, 0.0
        tgt = min(target, math.radians(60))
        for _ in range(200):
            q, _ = o.step(q, np.array([[target]]))
            th = th + 2 * math.atan(w * 0.01 / 2)
            lim = min(max(th, math.radians(-90)), math.radians(60)) - th  # soft limit (R7, R8)
            w = w + ((20 * (tgt - th) + 1000 * lim) / 0.5) * 0.01
            r = q["rot"][0, 1]
            assert abs(2 * math.atan2(r[1], r[0]) - th) < 1e-11
            assert abs(q["ang"][0, 1, 0] - w) < 1e-11


def test_app_a_pendulum_period():
    """Small-angle period of the App. A pendulum:
    T = 2π√((I + mL²)/(mgL)) = 2.8384 s; within 1e-3 relative at h = 0.01."""
    o = oracle.Oracle(oracle.load_scene("appA"))
    th0 = 0.05
    q = qp1(o, pos=[[0, 0, 0], [0, math.sin(th0), -math.cos(th0)]],
            rot=[[1, 0, 0, 0], [math.cos(th0 / 2), math.sin(th0 / 2), 0, 0]])
    T_cf = 2 * math.pi * math.sqrt(2.0 / 9.8)
    assert abs(T_cf - cf("pendulum_period")) < 1e-4
    ys, t = [], []
    for n in range(1200):
        q, _ = o.step(q)
        ys.append(q["pos"][0, 1, 1])
        t.append((n + 1) * 0.01)
    ys = np.array(ys)
    # downward zero crossings, linearly interpolated
    idx = np.where((ys[:-1] > 0) & (ys[1:] <= 0))[0]
    tc = [t[i] + (t[i + 1] - t[i]) * ys[i] / (ys[i] - ys[i + 1]) for i in idx]
    period = np.mean(np.diff(tc))
    assert abs(period - T_cf) / T_cf < 1e-3


def momentum_scene():
    """A 5-body free-floating chain: no gravity, no colliders, no damping, isotropic
    inertia, 1- 2- and 3-dof joints with torque actuators (Fig. 5 protocol)."""
    bodies = "\n".join(f'bodies {{ name: "L{i}" mass: {1 + 0.5 * i} inertia {{ x: {0.3 + 0.1 * i} y: {0.3 + 0.1 * i} z: {0.3 + 0.1 * i} }} }}'
                       for i in range(5))
    lims = ["angle_limit { min: -60 max: 60 }",
            "angle_limit { min: -45 max: 30 } angle_limit { min: -20 max: 20 }",
            "angle_limit { min: -80 max: 10 } angle_limit { min: -20 max: 20 } angle_limit { min: -30 max: 30 }",
            "angle_limit { min: 10 max: 70 }"]
    joints = "\n".join(
        f'joints {{ name: "J{i}" parent: "L{i}" child: "L{i + 1}" stiffness: 800 '
        f'parent_offset {{ x: 0.3 y: 0.05 }} child_offset {{ x: -0.25 z: 0.02 }} '
        f'rotation {{ z: {20 * i} y: 10 }} {lims[i]} }}' for i in range(4))
    acts = "\n".join(f'actuators {{ name: "A{i}" joint: "J{i}" strength: 0.5 torque {{}} }}' for i in range(4))
    return f"dt: 0.01 substeps: 2\n{bodies}\n{joints}\n{acts}\n"


def momenta(o, q):
    m = np.array([b.mass for b in o.sys.bodies])
    I = np.array([b.inertia[0] for b in o.sys.bodies])
    P = (m[None, :, None] * q["vel"]).sum(1)
    L = (np.cross(q["pos"], m[None, :, None] * q["vel"]) + I[None, :, None] * q["ang"]).sum(1)
    return P, L


def test_momentum_conservation_random_torques():
    """Newton's third law per joint/actuator ⇒ linear momentum exactly constant;
    isotropic inertia + no damping ⇒ angular momentum exactly constant (R4, R5;
    SPEC.md:248-249; 'exceptionally well')."""
    o = oracle.Oracle(momentum_scene())
    n = 8
    q = o.batch_default_qp(n)
    rng = np.random.default_rng(0)
    q["vel"] += rng.uniform(-1, 1, q["vel"].shape)
    q["ang"] += rng.uniform(-1, 1, q["ang"].shape)
    P0, L0 = momenta(o, q)
    for _ in range(100):
        q, ex = o.step(q, rng.uniform(-1, 1, (n, o.act_dim)))
    P1, L1 = momenta(o, q)
    assert np.max(np.abs(P1 - P0)) < 1e-12 * (1 + np.max(np.abs(P0)))
    assert np.max(np.abs(L1 - L0)) < 1e-11 * (1 + np.max(np.abs(L0)))


def test_newton_third_law_single_step():
    """Σ m·Δv over a jointed pair = 0 for any displacement."""
    o = oracle.Oracle(momentum_scene())
    q = o.batch_default_qp(4)
    rng = np.random.default_rng(3)
    q["pos"] += rng.normal(scale=0.05, size=q["pos"].shape)
    q["vel"] = rng.normal(size=q["vel"].shape)
    m = np.array([b.mass for b in o.sys.bodies])
    p0 = (m[None, :, None] * q["vel"]).sum(1)
    q1, _ = o.step(q, rng.uniform(-1, 1, (4, o.act_dim)))
    p1 = (m[None, :, None] * q1["vel"]).sum(1)
    assert np.max(np.abs(p1 - p0)) < 1e-12


# ---------------------------------------------------------------- contacts
def test_ball_drop_closed_forms():
    """Sphere–plane Baumgarte contact (R1, R13): first contact at substep 97 with
    d = g h²·97·96/2 − (z0 − r); rebound v = −gh + βd/h; rest depth d* = g h²/β;
    near rest the deviation decays by (1−β) per substep; z(1000) = r − d*."""
    o = oracle.Oracle(oracle.load_scene("ball"))
    q = o.batch_default_qp(1)
    g, h, beta, r, z0 = 9.8, 0.01, 0.2, 0.5, 5.0
    first = None
    traj = []
    for n in range(1, 1001):
        q, ex = o.step(q)
        traj.append(q["pos"][0, 1, 2])
        if first is None and ex["contact_active"][0, 0]:
            first = n
            d_cf = g * h * h * n * (n - 1) / 2 - (z0 - r)
            assert abs(d_cf - cf("ball_first_contact_d")) < 1e-12
            assert abs(q["vel"][0, 1, 2] - (-g * h + beta * d_cf / h)) < 1e-12
            assert abs(q["vel"][0, 1, 2] - cf("ball_rebound_v")) < 1e-4
    assert first == int(cf("ball_first_contact_substep"))
    dstar = g * h * h / beta
    assert abs(dstar - cf("ball_settle_d")) < 1e-12
    assert abs(traj[-1] - (r - dstar)) < 1e-12
    assert abs(traj[-1] - cf("ball_z_1000")) < 1e-12
    # geometric decay of the deviation from rest: δ_{n+1} = (1 − β)·δ_n
    dev = np.array(traj[700:720]) - (r - dstar)
    ok = np.abs(dev[:-1]) > 1e-13
    if ok.any():
        assert np.allclose(dev[1:][ok] / dev[:-1][ok], 1 - beta, atol=1e-6)


def test_rolling_ball_five_sevenths():
    """Coulomb friction impulse at the contact point conserves angular momentum
    about it, so a sliding solid sphere (I = 2/5 m r²) ends rolling at exactly
    v_f = 5/7·v0 (R13); sliding lasts ≈ 2v0/(7μg)."""
    o = oracle.Oracle(oracle.load_scene("ball"))
    dstar = 9.8 * 0.01 ** 2 / 0.2
    q = qp1(o, pos=[[0, 0, 0], [0, 0, 0.5 - dstar]], vel=[[0, 0, 0], [3.0, 0, 0]])
    slide_end = None
    for n in range(1, 101):
        q, _ = o.step(q)
        v, w = q["vel"][0, 1], q["ang"][0, 1]
        slip = v[0] - 0.5 * w[1]  # contact point velocity (ω × (0,0,−r))_x = −r·ω_y → v_x + ...
        if slide_end is None and abs(v[0] - 0.5 * w[1]) < 1e-12:
            slide_end = n
    assert abs(q["vel"][0, 1, 0] - 3.0 * 5 / 7) < 1e-12
    assert abs(q["vel"][0, 1, 0] - cf("rolling_vf")) < 1e-12
    assert slide_end == 9  # continuous estimate 2·3/(7·9.8)/0.01 = 8.7 substeps
    del slip


def box_scene(combine=""):
    return f"""dt: 0.01 gravity {{ z: -9.8 }} baumgarte_erp: 0.2
bodies {{ name: "G" frozen {{ all: true }} colliders {{ plane {{}} }} }}
bodies {{ name: "Cube" mass: 1 inertia {{ x: {2 / 3 * 0.25} y: {2 / 3 * 0.25} z: {2 / 3 * 0.25} }}
  colliders {{ box {{ halfsize {{ x: 0.5 y: 0.5 z: 0.5 }} }} }} }}
defaults {{ qps {{ name: "Cube" pos {{ z: 0.51 }} }} }}"""


@pytest.mark.parametrize("combine_sum", [False, True])
def test_resting_cube(combine_sum):
    """Uniform cube on a plane: k_n = 1/m + h_y²/I_x + h_x²/I_y = 4/m per corner; the
    mean of the 4 corner impulses (R14) settles at d* = g h² m k_n/β; the literal
    sum (test switch) at g h² m k_n/(4β) = g h²/β."""
    o = oracle.Oracle(box_scene(), combine_sum=combine_sum)
    q = o.batch_default_qp(1)
    for _ in range(600):
        q, ex = o.step(q)
    g, h, beta, m = 9.8, 0.01, 0.2, 1.0
    kn = 1 / m + 0.25 / (2 / 3 * 0.25) + 0.25 / (2 / 3 * 0.25)
    assert abs(kn - 4.0) < 1e-12
    dstar = g * h * h * m * kn / beta / (4 if combine_sum else 1)
    d = 0.5 - q["pos"][0, 1, 2]
    assert abs(d - dstar) < 1e-9
    assert list(ex["contact_active"][0]) == [1, 1, 1, 1, 0, 0, 0, 0]  # bottom corners (z bit = 0)


def capsule_scene(rot):
    return f"""dt: 0.01 gravity {{ z: -9.8 }}
bodies {{ name: "G" frozen {{ all: true }} colliders {{ plane {{}} }} }}
bodies {{ name: "Cap" mass: 2 inertia {{ x: 0.7 y: 0.7 z: 0.3 }}
  colliders {{ rotation {{ {rot} }} capsule {{ radius: 0.1 length: 1.0 }} }} }}
defaults {{ qps {{ name: "Cap" pos {{ z: 0.11 }} }} }}"""


def test_capsule_flat_and_vertical():
    """Capsule resting flat: both ends active, k_n = 1/m + ℓ²/I_⊥, d* = g h² m k_n/β.
    Vertical: one end active, k_n = 1/m, d* = g h²/β."""
    g, h, beta, m = 9.8, 0.01, 0.2, 2.0
    o = oracle.Oracle(capsule_scene("y: 90"))
    q = o.batch_default_qp(1)
    for _ in range(800):
        q, ex = o.step(q)
    ell = 0.5 - 0.1
    kn = 1 / m + ell ** 2 / 0.7
    assert abs((0.1 - q["pos"][0, 1, 2]) - g * h * h * m * kn / beta) < 1e-9
    assert list(ex["contact_active"][0]) == [1, 1]
    o = oracle.Oracle(capsule_scene("x: 0").replace("z: 0.11", "z: 0.51"))
    q = o.batch_default_qp(1)
    for _ in range(800):
        q, ex = o.step(q)
    assert abs((0.5 - q["pos"][0, 1, 2]) - g * h * h / beta) < 1e-9
    assert list(ex["contact_active"][0]) == [0, 1]  # slot 1 = the lower end c − ℓâ


def _seg_points(c, axis, ell, k):
    t = np.linspace(-1, 1, k)
    return c[None, :] + (ell * t)[:, None] * axis[None, :]


def _quat_to_axis(q):
    w, x, y, z = q
    return np.array([2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)])


@pytest.mark.parametrize("seed", range(6))
def test_capsule_capsule_distance_brute_force(seed):
    """Closest distance between capsule segments (Ericson §5.1.9) vs brute force over
    4000 × 4000 samples: d = r_A + r_B − min |p − q|."""
    txt = """dt: 0.01
bodies { name: "A" colliders { capsule { radius: 0.1 length: 1.2 } } }
bodies { name: "B" colliders { capsule { radius: 0.15 length: 0.8 } } }
collide_include { first: "A" second: "B" }"""
    o = oracle.Oracle(txt)
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-0.4, 0.4, (2, 3))
    rot = rng.normal(size=(2, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    d, n, pt, par = o.slot_geometry(0, pos, rot)
    k = 4000
    pa = _seg_points(pos[0], _quat_to_axis(rot[0]), 0.5, k)
    pb = _seg_points(pos[1], _quat_to_axis(rot[1]), 0.25, k)
    dmin = np.inf
    for i in range(0, k, 500):
        dd = np.linalg.norm(pa[i:i + 500, None, :] - pb[None, :, :], axis=-1)
        dmin = min(dmin, dd.min())
    d_bf = 0.25 - dmin
    # sampled distances are never below the exact minimum, and exceed it by at most
    # the sampling step (1.2/(k−1) along A plus 0.8/(k−1) along B)
    assert d >= d_bf - 1e-12
    assert d <= d_bf + 2.0 / (k - 1)
    assert abs(np.linalg.norm(n) - 1) < 1e-12


def test_capsule_capsule_perpendicular_crossing():
    """Perpendicular crossing → midpoints; d = r_A + r_B − separation (textbook)."""
    txt = """dt: 0.01
bodies { name: "A" colliders { rotation { y: 90 } capsule { radius: 0.1 length: 1.2 } } }
bodies { name: "B" colliders { rotation { x: 90 } capsule { radius: 0.15 length: 0.8 } } }
collide_include { first: "A" second: "B" }"""
    o = oracle.Oracle(txt)
    pos = np.array([[0, 0, 0.2], [0, 0, 0.0]])
    rot = np.array([[1.0, 0, 0, 0], [1.0, 0, 0, 0]])
    d, n, pt, par = o.slot_geometry(0, pos, rot)
    assert abs(d - (0.25 - 0.2)) < 1e-12
    assert np.allclose(n, [0, 0, 1], atol=1e-12)
    assert np.allclose(pt, [0, 0, 0.5 * ((0.2 - 0.1) + (0.0 + 0.15))], atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_sphere_capsule_distance_brute_force(seed):
    txt = """dt: 0.01
bodies { name: "S" colliders { sphere { radius: 0.2 } } }
bodies { name: "C" colliders { capsule { radius: 0.1 length: 1.0 } } }
collide_include { first: "C" second: "S" }"""
    o = oracle.Oracle(txt)
    assert o.sys.slot_table()[0, 1] == 4  # sphere_capsule, sphere oriented as A
    assert o.sys.slot_table()[0, 2] == 0
    rng = np.random.default_rng(seed)
    pos = rng.uniform(-0.5, 0.5, (2, 3))
    rot = rng.normal(size=(2, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    d, n, pt, _ = o.slot_geometry(0, pos, rot)
    k = 200001
    pb = _seg_points(pos[1], _quat_to_axis(rot[1]), 0.4, k)
    dmin = np.linalg.norm(pb - pos[0][None, :], axis=1).min()
    assert abs(d - (0.3 - dmin)) < 1e-9


def test_sphere_sphere_geometry():
    """Sphere–sphere: d = r_A + r_B − |c_A − c_B|, n from B to A, contact point at the
    midpoint of the two surface points (R18); coincident centres → n = ẑ (R16)."""
    txt = """dt: 0.01
bodies { name: "A" colliders { position { x: 0.1 } sphere { radius: 0.3 } } }
bodies { name: "B" colliders { sphere { radius: 0.2 } } }"""
    o = oracle.Oracle(txt)
    assert o.sys.slot_table().tolist() == [[0, 3, 0, 1, 0, 1, 0]]
    rng = np.random.default_rng(4)
    for _ in range(20):
        pos = rng.uniform(-0.3, 0.3, (2, 3))
        rot = rng.normal(size=(2, 4))
        rot /= np.linalg.norm(rot, axis=1, keepdims=True)
        ca = pos[0] + _rotate(rot[0], [0.1, 0, 0])
        cb = pos[1]
        dist = np.linalg.norm(ca - cb)
        d, n, pt, _ = o.slot_geometry(0, pos, rot)
        assert abs(d - (0.5 - dist)) < 1e-12
        assert np.allclose(n, (ca - cb) / dist, atol=1e-12)
        assert np.allclose(pt, 0.5 * ((ca - 0.3 * n) + (cb + 0.2 * n)), atol=1e-12)
    d, n, pt, _ = o.slot_geometry(0, np.array([[-0.1, 0, 0], [0, 0, 0.0]]), np.array([[1.0, 0, 0, 0]] * 2))
    assert abs(d - 0.5) < 1e-12 and np.allclose(n, [0, 0, 1])


def _rotate(q, v):
    from scipy.spatial.transform import Rotation
    return Rotation.from_quat([q[1], q[2], q[3], q[0]]).apply(v)


def test_sphere_plane_examples():
    """r 0.5 at z 0.6 → no contact; at z 0.4 → d = 0.1, n = +z."""
    o = oracle.Oracle(oracle.load_scene("ball"))
    rot = np.array([[1.0, 0, 0, 0], [1.0, 0, 0, 0]])
    d, n, pt, _ = o.slot_geometry(0, np.array([[0, 0, 0], [0, 0, 0.6]]), rot)
    assert d < 0
    d, n, pt, _ = o.slot_geometry(0, np.array([[0, 0, 0], [0, 0, 0.4]]), rot)
    assert abs(d - 0.1) < 1e-12 and np.allclose(n, [0, 0, 1]) and np.allclose(pt, [0, 0, -0.1])


# ---------------------------------------------------------------- whole-step invariants
@pytest.mark.parametrize("scene", ["ant", "humanoid", "halfcheetah", "grasp", "fetch"])
def test_scene_independence_and_determinism(scene):
    """Stepping a batch equals stepping each env alone, bitwise."""
    o = oracle.Oracle(oracle.load_scene(scene))
    n = 6
    q = o.reset(n, 7, 0.1, 0.1)
    rng = np.random.default_rng(0)
    for _ in range(3):
        q, _ = o.step(q, rng.uniform(-1, 1, (n, o.act_dim)))
    a = rng.uniform(-1, 1, (n, o.act_dim))
    qa, exa = o.step(q, a)
    qb, exb = o.step(q, a, threads=3)
    for i in range(n):
        qi, exi = o.step({k: v[i:i + 1] for k, v in q.items()}, a[i:i + 1])
        for k in qa:
            assert np.array_equal(qi[k][0], qa[k][i])
        assert np.array_equal(exi["contact_active"][0], exa["contact_active"][i])
    for k in qa:
        assert np.array_equal(qa[k], qb[k])


def test_philox_known_answers():
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as f:
        rows = [l.split() for l in f if l.strip() and not l.startswith("#")]
    for r in rows:
        v = [int(x, 16) for x in r]
        assert philox4x32_10(v[0:4], v[4:6]) == v[6:10]


def test_reset_noise_range_and_masks():
    o = oracle.Oracle(oracle.load_scene("halfcheetah"))
    q = o.reset(64, 123, 0.1, 0.2)
    d = o.default_qp()
    dv = q["vel"] - d["vel"][None]
    dw = q["ang"] - d["ang"][None]
    assert np.all(np.abs(dv) <= 0.1) and np.all(np.abs(dw) <= 0.2)
    assert np.all(dv[:, :, 1] == 0) and np.all(dw[:, :, [0, 2]] == 0)  # planar masks
    assert np.all(dv[:, 0] == 0)  # static ground
    assert np.array_equal(q["pos"], np.broadcast_to(d["pos"], q["pos"].shape))
    assert np.std(dv[:, 1:, 0]) > 0.04  # U(−0.1, 0.1) has σ ≈ 0.0577


def test_op_counts_ant():
    """Algorithmic flop count per ant env-step (SURVEY §8(d) estimate ≈ 58 k)."""
    o = oracle.Oracle(oracle.load_scene("ant"))
    q = o.reset(4, 0, 0.1, 0.1)
    fl, mu = o.count_ops(q, np.zeros((4, 8)))
    per = fl / 4
    assert 30e3 < per < 90e3
    assert mu > 0


def test_random_action_stream():
    """NEXT-2 action generator: values in [−1, 1) on the 2⁻²³ grid, the counter
    layout (env, step, k // 4, tag) of the header, distinct per env and step,
    and a disjoint counter space from the reset noise (tag word)."""
    from oracle.philox import ACT_TAG, random_actions, uniform_pm1
    a = random_actions(5, 6, 3, seed=2 ** 40 + 7, env_offset=10, step0=100)
    assert a.shape == (3, 5, 6) and np.all(a >= -1) and np.all(a < 1)
    assert np.array_equal(a * 2 ** 23, np.round(a * 2 ** 23))
    key = ((2 ** 40 + 7) & 0xFFFFFFFF, (2 ** 40 + 7) >> 32)
    x = philox4x32_10((12, 101, 1, ACT_TAG), key)
    assert a[1, 2, 4] == uniform_pm1(x[0]) and a[1, 2, 5] == uniform_pm1(x[1])
    assert len(np.unique(a.reshape(-1))) == a.size
    b = random_actions(5, 6, 3, seed=2 ** 40 + 7, env_offset=11, step0=100)
    assert np.array_equal(a[:, 1:], b[:, :-1])  # env ids are global
