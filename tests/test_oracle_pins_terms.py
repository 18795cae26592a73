"""Closed-form pins of individual oracle terms that the whole-motion pins in
test_oracle_pins.py leave free (VERDICT r1 "What's weak" 1): the TORQUE
actuator and its clamp (R11), the elasticity term of the
contact law (R13), the friction coefficient μ (R13), the world
inverse inertia of a rotated anisotropic body (R4, App. A `inertia {x y z}`,
PAPER.md:332) and the op counter behind the roofline numerator (SURVEY §8(d)
counting convention).  Each expected value is derived from the mechanics of the
discrete map in the docstring, not re-typed from the oracle's code; DESIGN.md §9
records the mutation runs each of these tests catches.  CPU only.
"""
import math

import numpy as np
import pytest

import oracle


def qp1(o, **kw):
    q = o.batch_default_qp(1)
    for k, v in kw.items():
        q[k][0] = v
    return q


# ---------------------------------------------------------------- TORQUE actuator (R11)
def torque_pair(rotation="", strength=3.0, Ip=2.0, Ic=0.5):
    """Two free bodies (no gravity, no colliders) joined at a common anchor by a hinge
    with wide limits and a TORQUE actuator: in the default pose the anchors coincide
    (linear spring force 0) and the joint angles are 0 (no limit/alignment torque)."""
    return f"""dt: 0.01 substeps: 1
bodies {{ name: "P" mass: 1 inertia {{ x: {Ip} y: {Ip} z: {Ip} }} }}
bodies {{ name: "C" mass: 1 inertia {{ x: {Ic} y: {Ic} z: {Ic} }} }}
joints {{ name: "J" parent: "P" child: "C" stiffness: 1000 {rotation}
  parent_offset {{ z: -0.5 }} child_offset {{ z: 0.5 }} angle_limit {{ min: -170 max: 170 }} }}
actuators {{ name: "A" joint: "J" strength: {strength} torque {{}} }}"""


@pytest.mark.parametrize("a", [0.6, -0.25, 2.5, -3.0])
def test_torque_actuator_single_substep(a):
    """From rest, one substep of a hinge TORQUE actuator changes the angular velocities by
    Δω_child = +s·clamp(a, −1, 1)·h/I_c and Δω_parent = −s·clamp(a, −1, 1)·h/I_p about the
    hinge axis (x̂ of the joint frame), Newton's third law; |a| > 1 exercises the clamp."""
    s, h, Ip, Ic = 3.0, 0.01, 2.0, 0.5
    o = oracle.Oracle(torque_pair(strength=s, Ip=Ip, Ic=Ic))
    q, _ = o.step(o.batch_default_qp(1), np.array([[a]]))
    tau = s * max(-1.0, min(1.0, a))
    assert np.allclose(q["ang"][0, 1], [tau * h / Ic, 0, 0], atol=1e-15, rtol=1e-14)
    assert np.allclose(q["ang"][0, 0], [-tau * h / Ip, 0, 0], atol=1e-15, rtol=1e-14)
    assert np.all(q["vel"] == 0)


def test_torque_actuator_axis_follows_joint_rotation():
    """The free axis is the joint frame's x̂ = rotate(rotation, x̂): a joint rotated by 90°
    about z (App. A `rotation`) drives the child about world ŷ."""
    s, h, Ic = 3.0, 0.01, 0.5
    o = oracle.Oracle(torque_pair(rotation="rotation { z: 90 }", strength=s, Ic=Ic))
    q, _ = o.step(o.batch_default_qp(1), np.array([[0.4]]))
    assert np.allclose(q["ang"][0, 1], [0, s * 0.4 * h / Ic, 0], atol=1e-15)


def test_torque_actuator_constant_spin_up():
    """Frozen parent, child hinged at its own centre (child_offset 0): a constant torque
    a·s makes ω_x grow by exactly s·clamp(a)·h/I per substep (ω_n = n·s·a·h/I) while
    the hinge angle advances by 2·atan(ω h/2) per substep (R3)."""
    s, h, I = 2.0, 0.01, 0.8
    txt = f"""dt: {h}
bodies {{ name: "P" frozen {{ all: true }} }}
bodies {{ name: "C" mass: 1 inertia {{ x: {I} y: {I} z: {I} }} }}
joints {{ name: "J" parent: "P" child: "C" stiffness: 1000 angle_limit {{ min: -180 max: 180 }} }}
actuators {{ name: "A" joint: "J" strength: {s} torque {{}} }}"""
    o = oracle.Oracle(txt)
    q = o.batch_default_qp(1)
    th = 0.0
    for n in range(1, 60):
        q, _ = o.step(q, np.array([[1.7]]))   # clamped to 1
        th = th + 2 * math.atan((n - 1) * s * h / I * h / 2)
        assert abs(q["ang"][0, 1, 0] - n * s * h / I) < 1e-12
        r = q["rot"][0, 1]
        assert abs(2 * math.atan2(r[1], r[0]) - th) < 1e-12


# ---------------------------------------------------------------- elasticity e (R13)
def ball_text(e=0.0, mu=1.0, gravity=-9.8):
    return f"""dt: 0.01 substeps: 1 gravity {{ z: {gravity} }}
friction: {mu} elasticity: {e} baumgarte_erp: 0.2
bodies {{ name: "G" frozen {{ all: true }} colliders {{ plane {{}} }} }}
bodies {{ name: "Ball" mass: 1 inertia {{ x: 0.1 y: 0.1 z: 0.1 }} colliders {{ sphere {{ radius: 0.5 }} }} }}"""


@pytest.mark.parametrize("e", [0.0, 0.5, 1.0])
def test_elastic_rebound_single_substep(e):
    """A ball (no gravity) hitting the plane at u⁻ = −2 m/s with penetration d after the
    kinematic step: the lever arm r×n is 0, so k(n) = 1/m and the impulse law
    j_n = (−(1+e)u⁻ + βd/h)/k(n) gives the post-impact velocity v⁺ = −e·u⁻ + βd/h."""
    o = oracle.Oracle(ball_text(e=e, gravity=0.0))
    h, beta, r = 0.01, 0.2, 0.5
    z0, u = 0.51, -2.0
    q = qp1(o, pos=[[0, 0, 0], [0, 0, z0]], vel=[[0, 0, 0], [0, 0, u]])
    q, ex = o.step(q)
    d = r - (z0 + h * u)
    assert abs(q["vel"][0, 1, 2] - (-e * u + beta * d / h)) < 1e-12
    assert ex["contact_active"][0, 0] == 1


def test_elastic_drop_bounces_to_e_squared_height():
    """Dropped from rest, a ball with e = 0.8 leaves its first bounce with about e times
    its impact speed (the Baumgarte term adds βd/h, small at this height), so the
    apex of the first bounce is ≈ e²·(drop height) above the contact surface; with
    e = 0 it stays within the Baumgarte pop-up of the rest depth."""
    for e, lo, hi in ((0.8, 0.8 ** 2 * 0.85, 0.8 ** 2 * 1.15), (0.0, -0.01, 0.02)):
        o = oracle.Oracle(ball_text(e=e))
        q = qp1(o, pos=[[0, 0, 0], [0, 0, 1.5]])
        zs = []
        for _ in range(400):
            q, _ = o.step(q)
            zs.append(q["pos"][0, 1, 2])
        zs = np.array(zs)
        first = int(np.argmax(np.diff(zs) > 0))          # the first substep moving up
        apex = zs[first:first + 150].max() - 0.5
        assert lo < apex < hi, (e, apex)


# ---------------------------------------------------------------- friction μ (R13)
@pytest.mark.parametrize("mu", [0.3, 0.55, 1.0])
def test_sliding_ball_friction_saturated(mu):
    """A solid ball (I = 2/5·m·r²) sliding at v0 while resting at the equilibrium depth
    d* = g h²/β: the normal impulse per substep is exactly m·g·h, and while it slips the
    Coulomb-saturated friction impulse μ·m·g·h gives v_x(n) = v0 − n·μ·g·h and
    r·ω_y(n) = n·μ·g·h·(m r²/I) = 2.5·n·μ·g·h, so the slip v_x − r·ω_y shrinks by
    3.5·μ·g·h per substep; sliding ends in substep ⌈v0/(3.5 μ g h)⌉ with v = 5/7·v0."""
    g, h, beta, r, v0 = 9.8, 0.01, 0.2, 0.5, 3.0
    o = oracle.Oracle(ball_text(mu=mu))
    dstar = g * h * h / beta
    q = qp1(o, pos=[[0, 0, 0], [0, 0, r - dstar]], vel=[[0, 0, 0], [v0, 0, 0]])
    n_end = math.ceil(v0 / (3.5 * mu * g * h))
    for n in range(1, n_end + 5):
        q, _ = o.step(q)
        vx, wy = q["vel"][0, 1, 0], q["ang"][0, 1, 1]
        if n < n_end:
            assert abs(vx - (v0 - n * mu * g * h)) < 1e-12
            assert abs(r * wy - 2.5 * n * mu * g * h) < 1e-12
            assert vx - r * wy > 0
        else:
            assert abs(vx - r * wy) < 1e-12          # rolling
            assert abs(vx - 5.0 / 7.0 * v0) < 1e-12


# ---------------------------------------------------------------- rotated anisotropic I_w⁻¹ (R4)
def aniso_oscillator(k_l=300.0):
    """Frozen parent, hinge about world x̂; the child has body-frame inertia (1, 2, 3) and is
    oriented by Rz(−90°), which maps its local ŷ onto world x̂.  reference_rotation equal
    to that orientation makes it the hinge's zero angle (J_c = conj(Rf)⊗rotation)."""
    return f"""dt: 0.01
bodies {{ name: "P" frozen {{ all: true }} }}
bodies {{ name: "C" mass: 1 inertia {{ x: 1 y: 2 z: 3 }} }}
joints {{ name: "J" parent: "P" child: "C" stiffness: 1000 limit_stiffness: {k_l}
  reference_rotation {{ z: -90 }} angle_limit {{ min: 0 max: 0 }} }}"""


def test_rotated_anisotropic_inertia_torsional_oscillator():
    """About world x̂ the child's moment of inertia is its body-frame I_y = 2 (local ŷ lies on
    the hinge axis), so the hinge angle follows the torsional recurrence with I_y:
    θ_{n+1} = θ_n + 2·atan(ω_n h/2), ω_{n+1} = ω_n − (k_l/I_y)·θ_{n+1}·h, the rotation stays
    about x̂, and the period is 2π√(I_y/k_l) (not that of I_x = 1 or I_z = 3)."""
    from scipy.spatial.transform import Rotation
    k_l, Iy, h = 300.0, 2.0, 0.01
    o = oracle.Oracle(aniso_oscillator(k_l))
    q0 = o.batch_default_qp(1)
    rf = Rotation.from_euler("z", -90, degrees=True)
    xyzw = rf.as_quat()
    assert np.allclose(q0["rot"][0, 1], [xyzw[3], *xyzw[:3]], atol=1e-15)  # default_qp = Rf
    assert np.allclose(rf.apply([0, 1, 0]), [1, 0, 0], atol=1e-15)
    q = qp1(o, ang=[[0, 0, 0], [0.6, 0, 0]])
    th, w = 0.0, 0.6
    zs = []
    for n in range(400):
        q, _ = o.step(q)
        th = th + 2 * math.atan(w * h / 2)
        w = w - (k_l / Iy) * th * h
        assert abs(q["ang"][0, 1, 0] - w) < 1e-11
        assert abs(q["ang"][0, 1, 1]) < 1e-12 and abs(q["ang"][0, 1, 2]) < 1e-12
        rel = (Rotation.from_quat([*q["rot"][0, 1, 1:], q["rot"][0, 1, 0]]) * rf.inv()).as_rotvec()
        assert abs(rel[0] - th) < 1e-10 and abs(rel[1]) < 1e-12 and abs(rel[2]) < 1e-12
        zs.append(rel[0])
    zs = np.array(zs)
    up = np.where((zs[:-1] < 0) & (zs[1:] >= 0))[0]
    tc = [(i + 1 + (-zs[i]) / (zs[i + 1] - zs[i])) * h for i in up]
    period = float(np.mean(np.diff(tc)))
    assert abs(period - 2 * math.pi * math.sqrt(Iy / k_l)) < 0.01 * period
    for other in (1.0, 3.0):
        assert abs(period - 2 * math.pi * math.sqrt(other / k_l)) > 0.1 * period


def test_rotated_anisotropic_inertia_single_torque_axes():
    """A body with body-frame inertia (1, 2, 3) oriented by R_f (its default pose: App. A
    `reference_rotation`), driven for one substep by a pure torque τ about the hinge axis
    R_j·x̂ (TORQUE actuator, parent frozen, anchors at the child's centre, joint angle 0):
    Δω = R_f·diag(1/I)·R_fᵀ·τ·h — the inverse inertia tensor in world axes, computed here
    from scipy's rotation matrices.  R_j ≠ R_f, so τ is not along a principal axis and Δω
    is not parallel to τ."""
    from scipy.spatial.transform import Rotation
    s, h, a = 2.0, 0.01, 0.7
    ej, ef = [30, -50, 70], [10, 40, -60]
    txt = f"""dt: {h}
bodies {{ name: "P" frozen {{ all: true }} }}
bodies {{ name: "C" mass: 1 inertia {{ x: 1 y: 2 z: 3 }} }}
joints {{ name: "J" parent: "P" child: "C" stiffness: 1000
  rotation {{ x: {ej[0]} y: {ej[1]} z: {ej[2]} }} reference_rotation {{ x: {ef[0]} y: {ef[1]} z: {ef[2]} }}
  angle_limit {{ min: -90 max: 90 }} }}
actuators {{ name: "A" joint: "J" strength: {s} torque {{}} }}"""
    o = oracle.Oracle(txt)
    q0 = o.batch_default_qp(1)
    # intrinsic X-Y-Z Euler angles (the scene convention) == scipy "XYZ"
    Rj = Rotation.from_euler("XYZ", ej, degrees=True)
    Rf = Rotation.from_euler("XYZ", ef, degrees=True)
    # default_qp: child rotation = J ⊗ E(0) ⊗ conj(J) ⊗ Rf = Rf
    xyzw = Rf.as_quat()
    assert np.allclose(q0["rot"][0, 1], [xyzw[3], *xyzw[:3]], atol=1e-12)
    q, _ = o.step(q0, np.array([[a]]))
    tau_w = s * a * Rj.apply([1.0, 0, 0])
    Mf = Rf.as_matrix()
    expect = Mf @ np.diag([1.0, 0.5, 1 / 3]) @ Mf.T @ tau_w * h
    assert np.allclose(q["ang"][0, 1], expect, atol=1e-14), (q["ang"][0, 1], expect)
    assert not np.allclose(expect / np.linalg.norm(expect), tau_w / np.linalg.norm(tau_w), atol=1e-2)


# ---------------------------------------------------------------- op counter
# Convention: add/sub/mul 1 flop, FMA 2 (the oracle writes none: -ffp-contract=off), div and
# sqrt 4 flops + 1 MUFU, atan2/asin 20 flops + 1 MUFU; negation, comparison, min/max/clamp 0.
# Building blocks (every operand counted, including multiplications by exact 0/1 masks):
#   cross 9 (6 mul + 3 sub); dot 5 (3 mul + 2 add); qmul 28 (16 mul + 12 add/sub);
#   rotate(q, v) = v + w·t + u×t with t = 2·u×v: 9 + 3 + 3 + 9 + 6 = 30;
#   I_w⁻¹(q)·v = rotate(q, inv_rotate(q, v) ⊘ I): 30 + 3·4 + 30 = 72 flops, 3 MUFU.
KIN = 9 + (3 + 28 + 1 + 8 + 7 + 4 + 16)   # x += h⊙(M v) ; q = normalize(q + ½h (0, Mω)⊗q)
KIN_MUFU = 1 + 4                          # sqrt, 4 divisions
POT = (4 + 3 + 3 + 3 + 3 + 3) + (72 + 3 + 3 + 3)   # v: 1/m, (1/m)F, +g, h·, v+, mask | ω
POT_MUFU = 1 + 3
# sphere–plane narrowphase: c_A, c_B (rotate + add: 33 each), q_colA, q_colB (qmul 28 each),
# n = rotate(q_colB, ẑ) 30, d = r − (c − p0)·n: 3 + 5 + 1, pt = c − r n: 6
SPHERE_PLANE = 33 + 33 + 28 + 28 + 30 + 9 + 6
# active contact on one dynamic body A (B static):
#   rA, rB 3+3; u = (vA + ωA×rA) − (vB + ωB×rB) 27; u_n 5;
#   k(n) = 0 + 1/m + (r×n)·I_w⁻¹(r×n): 9 + 4 + 72 + 5 + 2 = 92 (4 MUFU);
#   j_n: (1+e) 1, ·u_n 1, β/h 4, ·d 1, + 1, /k 4 = 12 (2 MUFU); u_t 6; s_t = √(u_t·u_t) 9 (1);
#   P = j_n n 3; slipping: t̂ = (1/s_t) u_t 7 (1), k(t̂) 92 (4), s_t/k 4 (1), μ j_n 1, P −= j_t t̂ 6;
#   ΔV += (1/m)P 10 (1); ΔΩ += I_w⁻¹(rA×P) 9 + 72 + 3 = 84 (3)
CONTACT_ACTIVE = 6 + 27 + 5 + 92 + 12 + 6 + 9 + 3 + 10 + 84
CONTACT_ACTIVE_MUFU = 4 + 2 + 1 + 1 + 3
SLIP = 7 + 92 + 4 + 1 + 6
SLIP_MUFU = 1 + 4 + 1
COLLISION = 4 + 9 + 9          # 1/cnt, v += mask⊙(s ΔV), ω likewise
COLLISION_MUFU = 1
# hinge joint (dof 1) with a TORQUE actuator:
#   r_p, r_c 60; Δx 9; Δv 27; F = kΔx + c_l Δv 9; f_p, f_c, q_r 3·28; R02 4, R12 4, R22 5, R01 4,
#   R00 5; θ: 3·20 (3 MUFU); τ_0 = k_l(clamp − θ) 2, τ_1, τ_2 = −k_a θ 1 each; actuator s·clamp(a) + 2;
#   c1 = √(R12² + R22²) 7 (1); c0, s0 two divisions 8 (2); ic = c1/max(c1², .01) 5 (1);
#   b0 4, b2 2; τ_j = Σ τ_i b_i 15; τ_w = rotate(f_p, τ_j) 30; τ_d = c_a(ω_p − ω_c) 6;
#   child F 3, T 18 (+ (τ_w+τ_d) 3 + r_c×F 9 + 3 + ... ), parent F 3, T 18
HINGE_TORQUE = 60 + 9 + 27 + 9 + 84 + 22 + 60 + 4 + 2 + 7 + 8 + 5 + 6 + 15 + 30 + 6 + 3 + 18 + 3 + 18
HINGE_TORQUE_MUFU = 3 + 1 + 2 + 1


def test_op_count_ball_free_flight():
    """Ball scene, one substep in free flight: kinematic + sphere–plane narrowphase
    (inactive) + potential integrator of the one dynamic body = 343 flops, 9 MUFU."""
    o = oracle.Oracle(oracle.load_scene("ball"))
    assert KIN + SPHERE_PLANE + POT == 343
    fl, mu = o.count_ops(o.batch_default_qp(1))
    assert (fl, mu) == (KIN + SPHERE_PLANE + POT, KIN_MUFU + POT_MUFU)


def test_op_count_ball_sliding_contact():
    """Ball resting at d* and sliding: the active contact with its friction branch and the
    collision integrator on top of the free-flight substep = 729 flops, 27 MUFU."""
    o = oracle.Oracle(oracle.load_scene("ball"))
    dstar = 9.8 * 0.01 ** 2 / 0.2
    q = qp1(o, pos=[[0, 0, 0], [0, 0, 0.5 - dstar]], vel=[[0, 0, 0], [3.0, 0, 0]])
    fl, mu = o.count_ops(q)
    total = KIN + SPHERE_PLANE + POT + CONTACT_ACTIVE + SLIP + COLLISION
    assert total == 729
    assert (fl, mu) == (total, KIN_MUFU + POT_MUFU + CONTACT_ACTIVE_MUFU + SLIP_MUFU + COLLISION_MUFU)
    # without slip (at rest) the friction branch is skipped
    q = qp1(o, pos=[[0, 0, 0], [0, 0, 0.5 - dstar]])
    fl, mu = o.count_ops(q)
    assert fl == KIN + SPHERE_PLANE + POT + CONTACT_ACTIVE + COLLISION


def test_op_count_pendulum():
    """App. A pendulum + TORQUE actuator, one substep: the static parent is skipped by the
    integrators, so kinematic + one hinge with actuator + potential = 572 flops, 16 MUFU;
    per env-step × substeps (1)."""
    o = oracle.Oracle(oracle.load_scene("pendulum"))
    assert HINGE_TORQUE == 396
    fl, mu = o.count_ops(o.batch_default_qp(2), np.array([[0.3], [-2.0]]))
    assert (fl, mu) == (2 * (KIN + HINGE_TORQUE + POT), 2 * (KIN_MUFU + HINGE_TORQUE_MUFU + POT_MUFU))


def test_op_count_ant_is_the_sum_of_its_items():
    """Ant (9 dynamic bodies, 8 hinge+TORQUE joints, 1 sphere–plane + 8 capsule-end slots,
    S = 10): from a state with no contact active the count is exactly
    S·(9·(KIN + POT) + 8·HINGE_TORQUE + SPHERE_PLANE + 8·CAPSULE_END); a capsule end adds the
    axis rotate(q_colA, ẑ) 30, ℓ = ½L − r 2 and the end point c ± ℓâ 6 to the sphere case."""
    o = oracle.Oracle(oracle.load_scene("ant"))
    q = o.batch_default_qp(1)
    q["pos"][0, 1:, 2] += 3.0          # lifted: every slot inactive, joints still at rest pose
    S = o.sys.substeps
    capsule_end = SPHERE_PLANE + 30 + 2 + 6
    fl, mu = o.count_ops(q, np.zeros((1, 8)))
    assert fl == S * (9 * (KIN + POT) + 8 * HINGE_TORQUE + SPHERE_PLANE + 8 * capsule_end)
    assert mu == S * (9 * (KIN_MUFU + POT_MUFU) + 8 * HINGE_TORQUE_MUFU)


# ---------------------------------------------------------------- angular damping (R5, R6)
def test_damped_torsional_oscillator_recurrence():
    """Hinge with limits [0, 0] and angular damping c_a, frozen parent: the damping torque
    on the child is c_a·(ω_p − ω_c) = −c_a·ω_c (R5), so with the limit spring
    θ_{n+1} = θ_n + 2·atan(ω_n h/2), ω_{n+1} = ω_n − (k_l·θ_{n+1} + c_a·ω_n)·h/I."""
    txt = """dt: 0.01
bodies { name: "P" frozen { all: true } }
bodies { name: "C" mass: 1 inertia { x: 2 y: 2 z: 2 } }
joints { name: "J" parent: "P" child: "C" stiffness: 1000 limit_stiffness: 300 angular_damping: 4
  angle_limit { min: 0 max: 0 } }"""
    o = oracle.Oracle(txt)
    q = qp1(o, ang=[[0, 0, 0], [0.7, 0, 0]])
    th, w, h, I = 0.0, 0.7, 0.01, 2.0
    for _ in range(300):
        q, _ = o.step(q)
        th = th + 2 * math.atan(w * h / 2)
        w = w - (300 * th + 4 * w) * h / I
        r = q["rot"][0, 1]
        assert abs(2 * math.atan2(r[1], r[0]) - th) < 1e-12
        assert abs(q["ang"][0, 1, 0] - w) < 1e-12


# ---------------------------------------------------------------- contact Δv sums (brax_step_extras.contact_dp)
def test_contact_dp_resting_ball_is_g_dt():
    """A ball resting at its equilibrium depth d* = g h²/β with S substeps: in every substep
    the collision integrator adds exactly the velocity gravity removed, g·h upwards (the
    Baumgarte impulse βd*/h = g·h, u_n = 0), so Σ over the step's substeps of the collision
    integrator's Δv is (0, 0, S·g·h) = (0, 0, g·dt) and Δω = 0; the last substep's alone is g·h."""
    g, dt, S, beta, r = 9.8, 0.02, 4, 0.2, 0.5
    h = dt / S
    txt = f"""dt: {dt} substeps: {S} gravity {{ z: -{g} }} baumgarte_erp: {beta}
bodies {{ name: "G" frozen {{ all: true }} colliders {{ plane {{}} }} }}
bodies {{ name: "Ball" mass: 1 inertia {{ x: 0.1 y: 0.1 z: 0.1 }} colliders {{ sphere {{ radius: {r} }} }} }}"""
    o = oracle.Oracle(txt)
    q = qp1(o, pos=[[0, 0, 0], [0, 0, r - g * h * h / beta]])
    q, ex = o.step(q, contact_dv=True, contact_dp=True)
    assert np.allclose(ex["contact_dp"][0, 1], [0, 0, g * dt, 0, 0, 0], atol=1e-12)
    assert np.allclose(ex["contact_dv"][0, 1], [0, 0, g * h, 0, 0, 0], atol=1e-12)
    assert np.all(ex["contact_dp"][0, 0] == 0)       # static ground
    assert ex["contact_active"][0, 0] == S


def test_op_count_lean_convention_ball():
    """The lean convention (scene-neutral operations uncounted) for the free-flying ball:
    kinematic without the two unit-mask products (76 − 6), sphere–plane narrowphase without
    the zero collider offsets (2 × 33) and identity collider rotations (2 × 28) = 45, the
    potential integrator without its masks and with I_w⁻¹ of the isotropic ball as three
    products (16 + 9) = 140 flops; MUFU: kinematic 5 + 1/m = 6."""
    o = oracle.Oracle(oracle.load_scene("ball"))
    fl, mu = o.count_ops(o.batch_default_qp(1), lean=True)
    assert (KIN - 6) + (SPHERE_PLANE - 2 * 33 - 2 * 28) + (POT - 6 - 72 + 3) == 140
    assert (fl, mu) == (140, 6)
    assert o.count_ops(o.batch_default_qp(1)) == (343, 9)     # the default convention is unchanged
