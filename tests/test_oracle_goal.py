"""Pins of the goal-directed task (grasp / fetch; R36)
in the oracle's env epilogue: the progress reward against closed forms of free
motion, the hit bonus and marker placement against the Philox stream (itself pinned
by the Random123 known-answer vectors), the goal observation block against hand
positions, and the parser's checks."""
import math

import numpy as np
import pytest

import oracle
from oracle.env import Env
from oracle.philox import philox4x32_10, uniform_pm1

# A free ball in zero gravity (no contacts, no joints) and a frozen marker.
GOAL = """dt: 0.02
bodies {{ name: "Ball" mass: 1 inertia {{ x: 1 y: 1 z: 1 }} }}
bodies {{ name: "Target" mass: 1 inertia {{ x: 1 y: 1 z: 1 }} frozen {{ all: true }} {tcol} }}
defaults {{ qps {{ name: "Target" pos {{ x: 1 }} }} }}
task {{ torso: "Ball" survive_reward: 0.25 episode_length: {L}
  goal {{ object: "Ball" target: "Target" radius: 0.1 bonus: 5 range {{ x: 0.5 y: 0.25 z: 0 }} }} }}"""


def env(L=1000, tcol=""):
    return Env(oracle.Oracle(GOAL.format(L=L, tcol=tcol)))


def state(e, n, x, v):
    qp = e.o.batch_default_qp(n)
    qp["pos"][:, 0] = x
    qp["vel"][:, 0] = v
    return qp


def u3(env_id, body, field, episode, seed):
    x = philox4x32_10((env_id, body, field, episode), (seed & 0xFFFFFFFF, seed >> 32))
    return np.array([uniform_pm1(x[k]) for k in range(3)])


def test_goal_obs_dims_of_the_scenes():
    """grasp and fetch carry the goal block (R36): 11 + 2·Σdof + 9 + 6B."""
    for name, dof, B in (("grasp", 19, 17), ("fetch", 10, 12)):
        e = Env(oracle.Oracle(oracle.load_scene(name)))
        assert e.sys.act_dim == dof and len(e.sys.bodies) == B
        assert e.obs_dim == 11 + 2 * dof + 9 + 6 * B, name


def test_progress_reward_straight_at_the_marker():
    """Moving straight at the marker with speed v (no forces): d0 − d1 = v·dt, so the
    reward is v + survive (closed form of free flight)."""
    e = env()
    n = 4
    v = np.array([0.5, 1.0, 2.0, 3.0])
    qp = state(e, n, np.zeros(3), np.stack([v, 0 * v, 0 * v], 1))
    r = e.step(qp, np.zeros(n, np.int32), np.zeros(n, np.uint32), None, seed=1)
    assert np.allclose(r["reward"], v + 0.25, rtol=0, atol=1e-9)
    assert not r["done"].any()
    assert np.array_equal(r["qp"]["pos"][:, 1], np.tile([1.0, 0, 0], (n, 1)))  # no hit: the marker stays


def test_progress_reward_tangential_motion():
    """Moving across the line of sight (marker at distance 1, velocity ⟂): the distance
    grows to sqrt(1 + (v·dt)²); reward = (1 − sqrt(1 + (v·dt)²))/dt + survive."""
    e = env()
    v = 4.0
    qp = state(e, 1, np.zeros(3), np.array([0.0, v, 0.0]))
    r = e.step(qp, np.zeros(1, np.int32), np.zeros(1, np.uint32), None, seed=1)
    want = (1.0 - math.sqrt(1.0 + (v * 0.02) ** 2)) / 0.02 + 0.25
    assert abs(r["reward"][0] - want) < 1e-9


def test_hit_pays_the_bonus_and_places_the_marker_again():
    """Ending within the radius pays progress + bonus, and the marker moves to
    x̄ + range ⊙ u(env, T, 2 + steps', episode) (steps' = steps after this step)."""
    e = env()
    n, seed, off = 3, 77, 40
    qp = state(e, n, np.zeros(3), np.array([5.0, 0.0, 0.0]))  # x' = x + 0.1
    qp["pos"][:, 0, 0] = [0.85, 0.86, 0.5]  # d1 = 0.05, 0.04 (hits), 0.4 (misses)
    steps = np.array([0, 7, 0], np.int32)
    ep = np.array([3, 0, 0], np.uint32)
    r = e.step(qp, steps, ep, None, seed=seed, env_offset=off)
    d0 = 1.0 - qp["pos"][:, 0, 0]
    d1 = np.abs(1.0 - (qp["pos"][:, 0, 0] + 5.0 * 0.02))
    assert np.allclose(r["reward"], (d0 - d1) / 0.02 + 0.25 + 5.0 * np.array([1, 1, 0]), atol=1e-9)
    for i in (0, 1):
        want = np.array([1.0, 0.0, 0.0]) + np.array([0.5, 0.25, 0.0]) * u3(off + i, 1, 2 + steps[i] + 1, int(ep[i]), seed)
        assert np.allclose(r["qp"]["pos"][i, 1], want, atol=1e-15)
        assert np.all(np.abs(r["qp"]["pos"][i, 1] - [1, 0, 0]) <= [0.5, 0.25, 0.0])
    assert np.array_equal(r["qp"]["pos"][2, 1], [1.0, 0.0, 0.0])
    assert not np.array_equal(r["qp"]["pos"][0, 1], r["qp"]["pos"][1, 1])


def test_reset_places_the_marker_per_episode():
    """brax_env_reset places the marker from counter (env, T, 2, 0); the auto-reset of
    the k-th episode from (env, T, 2, k); z stays (range z = 0)."""
    e = env(L=1)
    seed = 5
    qp, steps, ep, obs = e.reset(4, seed, env_offset=10)
    for i in range(4):
        want = np.array([1.0, 0, 0]) + np.array([0.5, 0.25, 0]) * u3(10 + i, 1, 2, 0, seed)
        assert np.allclose(qp["pos"][i, 1], want, atol=1e-15)
    qp["pos"][:, 0] = [-3.0, 0, 0]  # far: no hit
    r = e.step(qp, steps, ep, None, seed=seed, env_offset=10)  # L = 1: every env is done
    assert r["done"].all() and np.array_equal(r["episode"], [1, 1, 1, 1])
    for i in range(4):
        want = np.array([1.0, 0, 0]) + np.array([0.5, 0.25, 0]) * u3(10 + i, 1, 2, 1, seed)
        assert np.allclose(r["qp"]["pos"][i, 1], want, atol=1e-15)
        assert r["qp"]["pos"][i, 1, 2] == 0.0


def test_goal_observation_block():
    """obs[11 + 2·Σdof : +9] = x_T − x_O, x_O − x_torso, v_O — hand-placed bodies."""
    txt = oracle.load_scene("fetch")
    e = Env(oracle.Oracle(txt))
    qp = e.o.batch_default_qp(1)
    g = e.task.goal
    qp["pos"][0, g.target] = [2.0, -1.0, 0.5]
    qp["pos"][0, e.task.torso] = [0.5, 0.25, 0.55]
    qp["vel"][0, e.task.torso] = [0.1, -0.2, 0.3]
    obs = e.observe(qp)
    k = 11 + 2 * e.sys.n_joint_dofs
    assert np.allclose(obs[0, k:k + 9], [1.5, -1.25, -0.05, 0, 0, 0, 0.1, -0.2, 0.3], atol=1e-15)
    # grasp: object (ball) and torso (palm) differ
    e = Env(oracle.Oracle(oracle.load_scene("grasp")))
    qp = e.o.batch_default_qp(1)
    g = e.task.goal
    qp["pos"][0, g.obj] = [0.1, 0.2, 0.3]
    qp["pos"][0, e.task.torso] = [0.0, 0.0, 0.5]
    qp["pos"][0, g.target] = [0.0, 0.0, 0.35]
    qp["vel"][0, g.obj] = [1.0, 2.0, 3.0]
    obs = e.observe(qp)
    k = 11 + 2 * e.sys.n_joint_dofs
    assert np.allclose(obs[0, k:k + 9], [-0.1, -0.2, 0.05, 0.1, 0.2, -0.2, 1, 2, 3], atol=1e-15)


@pytest.mark.parametrize("bad,where", [
    ('goal { object: "Ball" target: "Ball" radius: 0.1 }', "target"),       # not frozen
    ('goal { object: "Target" target: "Target" radius: 0.1 }', "object"),   # static object
    ('goal { object: "Ball" target: "Nope" radius: 0.1 }', "target"),
    ('goal { object: "Ball" target: "Target" }', "radius"),
    ('goal { object: "Ball" target: "Target" radius: 0 }', "radius"),
    ('goal { object: "Ball" target: "Target" radius: 0.1 range { x: -1 } }', "range"),
    ('goal { target: "Target" radius: 0.1 }', "object"),
    ('goal { object: "Ball" target: "Target" radius: 0.1 colour: 2 }', "colour"),
])
def test_goal_validation(bad, where):
    txt = GOAL.format(L=10, tcol="").split("task")[0] + 'task { torso: "Ball" ' + bad + " }"
    with pytest.raises(oracle.system.ValidationError, match=where):
        oracle.parse_system(txt)


def test_goal_marker_must_not_collide():
    with pytest.raises(oracle.system.ValidationError, match="collider"):
        env(tcol="colliders { sphere { radius: 0.1 } }")
