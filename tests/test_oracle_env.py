"""Pins of the oracle's env epilogue (NEXT-1, oracle/env.py): observation layout,
joint angles and rates, reward, done, auto-reset and contact observations,
each checked against something other than the oracle's own formula."""
import math
import os
import sys

import numpy as np
import pytest

import oracle
from oracle.env import Env
from oracle.philox import reset_qp

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
import astronaut  # noqa: E402  (independent numpy Euler extraction)


def env_of(text):
    return Env(oracle.Oracle(text))


TASK = """task {{ torso: "{torso}" {extra} }}"""


def test_table1_observation_dims():
    """Table 1: Ant obs 87, Halfcheetah obs 25 with our layout;
    act dims 8 and 7."""
    for name, obs, act in (("ant", 87, 8), ("halfcheetah", 25, 7)):
        e = env_of(oracle.load_scene(name))
        assert e.obs_dim == obs and e.sys.act_dim == act, name


def test_task_validation():
    base = oracle.load_scene("ball").split("defaults")[0]
    for bad in ('task { torso: "Nope" }', 'task { torso: "Ground" }', 'task { torso: "Ball" forward { } }',
                'task { torso: "Ball" healthy_z { min: 1 max: 0.5 } }', 'task { torso: "Ball" episode_length: 0 }',
                'task { torso: "Ball" ctrl_cost: -1 }', 'task { torso: "Ball" colour: 1 }'):
        with pytest.raises(oracle.system.ValidationError):
            oracle.parse_system(base + bad)


def test_free_body_observation_and_reward_closed_form():
    """A free body with no gravity: obs = (z, q, v, ω) exactly, and the forward
    reward (x' − x)·f/dt equals v·f (x' = x + v·dt), plus the survive reward."""
    txt = """dt: 0.02
bodies { name: "B" mass: 2 inertia { x: 1 y: 1 z: 1 } }
task { torso: "B" forward { x: 0.6 y: 0.8 } survive_reward: 0.25 }"""
    e = env_of(txt)
    assert e.obs_dim == 11
    qp = e.o.batch_default_qp(3)
    rng = np.random.default_rng(0)
    qp["pos"][:, 0] = rng.normal(size=(3, 3))
    qp["vel"][:, 0] = rng.normal(size=(3, 3))
    q = rng.normal(size=(3, 4))
    qp["rot"][:, 0] = q / np.linalg.norm(q, axis=1, keepdims=True)
    obs = e.observe(qp)
    assert np.array_equal(obs[:, 0], qp["pos"][:, 0, 2])
    assert np.array_equal(obs[:, 1:5], qp["rot"][:, 0])
    assert np.array_equal(obs[:, 5:8], qp["vel"][:, 0])
    r = e.step(qp, np.zeros(3, np.int32), np.zeros(3, np.uint32), None, seed=1)
    want = qp["vel"][:, 0] @ np.array([0.6, 0.8, 0.0]) + 0.25
    assert np.allclose(r["reward"], want, rtol=0, atol=1e-12)
    assert not r["done"].any() and np.array_equal(r["steps"], [1, 1, 1])


def test_ctrl_cost_is_the_only_action_dependence():
    """With a zero-strength actuator the dynamics ignore the action, so
    reward(a) − reward(0) = −ctrl_cost·‖a‖² exactly."""
    txt = oracle.load_scene("pendulum").replace("strength: 0.5", "strength: 0") + \
        'task { torso: "Child" ctrl_cost: 0.3 }'
    e = env_of(txt)
    qp = e.o.reset(4, 3, 0.1, 0.1)
    a = np.array([[0.5], [-1.0], [0.25], [2.0]])
    z = np.zeros((4,), np.int32)
    r1 = e.step(qp, z, z.view(np.uint32), a, seed=0)
    r0 = e.step(qp, z, z.view(np.uint32), np.zeros_like(a), seed=0)
    assert np.allclose(r1["reward"] - r0["reward"], -0.3 * a[:, 0] ** 2, rtol=0, atol=1e-12)


def test_hinge_angle_observation():
    """A hinge whose child is rotated by θ about the joint's x axis reads θ
    (the joint frame is rotated, so the hinge axis is not the world x)."""
    txt = """dt: 0.01
bodies { name: "P" frozen { all: true } }
bodies { name: "C" mass: 1 inertia { x: 1 y: 1 z: 1 } }
joints { name: "J" parent: "P" child: "C" stiffness: 100 rotation { z: 90 y: 20 } angle_limit { min: -170 max: 170 } }
task { torso: "C" }"""
    e = env_of(txt)
    j = e.sys.joints[0]
    for theta in (-2.5, -0.3, 0.0, 0.7, 1.9):
        qx = np.array([math.cos(theta / 2), math.sin(theta / 2), 0, 0])
        # child frame: q_c ⊗ J_c = J_p ⊗ Rx(θ)  ->  q_c = J_p ⊗ Rx(θ) ⊗ conj(J_c)
        jc = oracle.system.qmul(oracle.system.qconj(j.reference_rotation), j.rotation)
        qc = oracle.system.qmul(oracle.system.qmul(j.rotation, qx), oracle.system.qconj(jc))
        qp = e.o.batch_default_qp(1)
        qp["rot"][0, 1] = qc
        assert abs(e.observe(qp)[0, 5] - theta) < 1e-12


@pytest.mark.parametrize("scene", ["coverage", "humanoid"])
def test_joint_rates_are_the_time_derivative_of_the_angles(scene):
    """θ̇ (dual-basis projection of the relative angular velocity, R7) equals the
    central difference of θ, computed by an independent numpy extraction, along
    the exact free rotation q(t) = exp(t·ω/2)⊗q of every body."""
    e = env_of(oracle.load_scene(scene) + ('\ntask { torso: "Base" }' if scene == "coverage" else ""))
    qp = e.o.reset(16, 7, 0.0, 2.0)  # random body angular velocities
    rng = np.random.default_rng(1)
    q = qp["rot"] * 1.0
    for b in range(q.shape[1]):  # random orientations too
        r = rng.normal(size=(16, 4))
        q[:, b] = r / np.linalg.norm(r, axis=1, keepdims=True)
    qp["rot"] = q
    dof0 = 5
    obs = e.observe(qp)
    nq = e.sys.n_joint_dofs
    rates = obs[:, dof0 + nq + 6: dof0 + nq + 6 + nq]

    def advance(dt):
        w = qp["ang"]
        ang = np.linalg.norm(w, axis=-1, keepdims=True)
        axis = np.where(ang > 0, w / np.where(ang > 0, ang, 1), 0)
        dq = np.concatenate([np.cos(ang * dt / 2), np.sin(ang * dt / 2) * axis], -1)
        return astronaut.qmul(dq, qp["rot"])

    eps = 1e-6
    col = 0
    for j in e.sys.joints:
        th_p = astronaut.joint_angles(advance(eps)[:, j.parent], advance(eps)[:, j.child], j)
        th_m = astronaut.joint_angles(advance(-eps)[:, j.parent], advance(-eps)[:, j.child], j)
        fd = (th_p - th_m) / (2 * eps)
        for i in range(j.dof):
            ok = np.abs(np.cos(astronaut.joint_angles(qp["rot"][:, j.parent], qp["rot"][:, j.child], j)[:, 1])) > 0.2
            wrap = np.abs(th_p[:, i] - th_m[:, i]) < 1.0  # skip the ±π branch cut
            m = ok & wrap
            assert np.allclose(rates[m, col + i], fd[m, i], rtol=1e-5, atol=1e-5), (j.name, i)
        col += j.dof


def test_done_on_height_and_on_truncation():
    """Ball at z = 5 outside healthy_z [0.2, 1.0]: done after one step.  Ball
    resting at z = r − d* inside it: done exactly at episode_length (3)."""
    base = oracle.load_scene("ball")
    e = env_of(base + 'task { torso: "Ball" healthy_z { min: 0.2 max: 1.0 } episode_length: 3 }')
    z = np.zeros(2, np.int32)
    qp = e.o.batch_default_qp(2)
    r = e.step(qp, z, z.view(np.uint32), None, seed=5)
    assert r["done"].all() and np.array_equal(r["steps"], [0, 0]) and np.array_equal(r["episode"], [1, 1])
    dstar = 9.8 * 0.01 ** 2 / 0.2
    qp = e.o.batch_default_qp(2)
    qp["pos"][:, 1, 2] = 0.5 - dstar
    steps, ep = z.copy(), z.view(np.uint32).copy()
    for t in range(3):
        r = e.step(qp, steps, ep, None, seed=5)
        qp, steps, ep = r["qp"], r["steps"], r["episode"]
        assert bool(r["done"].all()) == (t == 2)
        assert r["x1_z"][0] == pytest.approx(0.5 - dstar, abs=1e-12) or t == 2


def test_auto_reset_draws_the_next_episode_counter():
    """A done env restarts from reset_qp with Philox counter (env id, b, f,
    episode + 1); episode 0 is brax_reset itself (Oracle.reset)."""
    e = env_of(oracle.load_scene("ant"))
    t = e.task
    qp0, steps, ep, obs0 = e.reset(6, seed=11, env_offset=100)
    ref = reset_qp(e.sys, e.o.default_qp(), 6, 11, t.reset_vel_noise, t.reset_ang_noise,
                   env_ids=100 + np.arange(6))
    for k in qp0:
        assert np.array_equal(qp0[k], ref[k])
    # env 0 of a plain brax_reset batch is env 0 here with env_offset 0
    plain = e.o.reset(3, 11, t.reset_vel_noise, t.reset_ang_noise)
    qpz, _, _, _ = e.reset(3, seed=11)
    for k in plain:
        assert np.array_equal(plain[k], qpz[k])
    steps = np.full(6, t.episode_length - 1, np.int32)  # truncation on this step
    ep = np.array([0, 1, 2, 3, 4, 5], np.uint32)
    a = np.zeros((6, e.sys.act_dim))
    r = e.step(qp0, steps, ep, a, seed=11, env_offset=100)
    assert r["done"].all() and np.array_equal(r["episode"], ep + 1) and not r["steps"].any()
    want = reset_qp(e.sys, e.o.default_qp(), 6, 11, t.reset_vel_noise, t.reset_ang_noise,
                    env_ids=100 + np.arange(6), episode=ep + 1)
    for k in want:
        assert np.array_equal(r["qp"][k], want[k])
    assert np.array_equal(r["obs"], e.observe(want))


def test_contact_observation_ball_drop():
    """At the first contact step n of the ball drop (R1, R13): the collision
    integrator changes v_z by βd/h + g·h·(n − 1) (the impulse cancels the
    pre-gravity velocity −g·h·(n−1) and adds the Baumgarte term); the obs holds
    it clipped to 1, zeros elsewhere."""
    e = env_of(oracle.load_scene("ball") + 'task { torso: "Ball" contact_obs: true }')
    assert e.obs_dim == 11 + 12
    g, h, beta, r0, z0 = 9.8, 0.01, 0.2, 0.5, 5.0
    qp = e.o.batch_default_qp(1)
    z = np.zeros(1, np.int32)
    for n in range(1, 200):
        res = e.step(qp, z, z.view(np.uint32), None, seed=0)
        qp = res["qp"]
        _, ex = None, None
        co = res["obs"][0, 11:].reshape(2, 6)
        if co[1, 2] != 0:
            d = g * h * h * n * (n - 1) / 2 - (z0 - r0)
            raw = beta * d / h + g * h * (n - 1)
            assert n == 97 and raw > 1
            assert co[1, 2] == 1.0 and np.all(co[1, [0, 1, 3, 4, 5]] == 0) and np.all(co[0] == 0)
            # unclipped value from the oracle step itself
            q2 = e.o.batch_default_qp(1)
            for _ in range(n - 1):
                q2, _ = e.o.step(q2)
            _, ex = e.o.step(q2, contact_dv=True)
            assert abs(ex["contact_dv"][0, 1, 2] - raw) < 1e-9
            break
    else:
        raise AssertionError("no contact")
