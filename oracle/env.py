"""Gym-like locomotion env epilogue on top of the oracle step (NEXT-1).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference may use this module.

What it computes (PAPER.md:105-122 "Gym-like environments", Table 1; :505-509
Ant / Humanoid rewards; SPEC.md:361-378 env_step / observe; R30-R35):

  observation of a QP (R32), one row per env:
    [ z_torso, q_torso (w, x, y, z),                     5
      θ: joint angles, joints by index, axes i < dof,     Σ dof
      v_torso, ω_torso,                                   6
      θ̇: joint rates, same order,                         Σ dof
      x_T − x_O, x_O − x_torso, v_O                       9 if task.goal (R36)
      clip(Δv_b, ±1), clip(Δω_b, ±1) for every body b ]   6B if task.contact_obs
  θ: the intrinsic X-Y-Z angles of q_r = conj(q_p⊗J_p)⊗(q_c⊗J_c), w ≥ 0 (R7);
  θ̇_i = b_i·ω_r with ω_r = R(q_p⊗J_p)ᵀ(ω_c − ω_p) and b the dual basis of the
  rotation axes (R7): the exact time derivative of θ;
  Δv_b, Δω_b: the collision integrator's velocity change of the step's last substep.

  reward (R31) = ((x'_torso − x_torso)·f)/dt + survive_reward − ctrl_cost·Σ_k a_k²
  goal tasks (R36; grasp / fetch): object O, frozen marker T,
    reward = (|x_O − x_T| − |x'_O − x_T|)/dt + survive_reward − ctrl_cost·Σ a² + bonus·hit,
    hit = |x'_O − x_T| < radius; a hit places the marker again at
    x̄_T + range ⊙ u(env, T, 2 + steps + 1, episode); every reset of episode k places it
    at x̄_T + range ⊙ u(env, T, 2, k) (u: the Philox reset-noise draw, x̄_T: default_qp).
  done (R33)   = z'_torso ∉ [min, max] (if healthy_z)  or  steps + 1 ≥ episode_length
  auto-reset (R34): a done env restarts from the task's reset noise with Philox
  counter (global env index, body, field, episode + 1); steps ← 0,
  episode ← episode + 1, contact obs ← 0.  reward / done describe the transition,
  obs the returned (possibly reset) state.
"""
from __future__ import annotations

import numpy as np

from .philox import philox4x32_10, reset_qp, uniform_pm1


def _qmul(a, b):
    aw, ax, ay, az = np.moveaxis(a, -1, 0)
    bw, bx, by, bz = np.moveaxis(b, -1, 0)
    return np.stack([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw], -1)


def _conj(q):
    return q * np.array([1.0, -1.0, -1.0, -1.0])


def _rotate(q, v):
    """R(q)·v for unit quaternions q [..., 4], v [..., 3]."""
    w, u = q[..., :1], q[..., 1:]
    t = 2.0 * np.cross(u, v)
    return v + w * t + np.cross(u, t)


def joint_angles_and_rates(sys, qp):
    """θ and θ̇ of every joint's free axes, [n, Σdof] each (R7)."""
    n = qp["pos"].shape[0]
    th_all, rate_all = [], []
    for j in sys.joints:
        jp = np.broadcast_to(j.rotation, (n, 4))
        jc = np.broadcast_to(_qmul(_conj(j.reference_rotation), j.rotation), (n, 4))
        fp = _qmul(qp["rot"][:, j.parent], jp)
        fc = _qmul(qp["rot"][:, j.child], jc)
        qr = _qmul(_conj(fp), fc)
        qr = np.where(qr[:, :1] < 0, -qr, qr)
        w, x, y, z = qr.T
        R02 = 2 * (x * z + w * y)
        R12 = 2 * (y * z - w * x)
        R22 = 1 - 2 * (x * x + y * y)
        R01 = 2 * (x * y - w * z)
        R00 = 1 - 2 * (y * y + z * z)
        th = np.stack([np.arctan2(-R12, R22), np.arcsin(np.clip(R02, -1, 1)), np.arctan2(-R01, R00)], -1)
        # dual basis of a0 = x, a1 = Rx(θ0)y, a2 = Rx(θ0)Ry(θ1)z in the parent joint frame (R7):
        # b0 = (1, s0 s1/c1, −c0 s1/c1), b1 = (0, c0, s0), b2 = (0, −s0/c1, c0/c1), 1/c1 guarded
        c1 = np.sqrt(R12 * R12 + R22 * R22)
        s1 = np.clip(R02, -1, 1)
        c0 = np.where(c1 > 0, R22 / np.where(c1 > 0, c1, 1), 1.0)
        s0 = np.where(c1 > 0, -R12 / np.where(c1 > 0, c1, 1), 0.0)
        ic = c1 / np.maximum(c1 * c1, 0.01)
        wr = _rotate(_conj(fp), qp["ang"][:, j.child] - qp["ang"][:, j.parent])
        rates = np.stack([wr[:, 0] + s0 * s1 * ic * wr[:, 1] - c0 * s1 * ic * wr[:, 2],
                          c0 * wr[:, 1] + s0 * wr[:, 2],
                          -s0 * ic * wr[:, 1] + c0 * ic * wr[:, 2]], -1)
        th_all.append(th[:, : j.dof])
        rate_all.append(rates[:, : j.dof])
    if not th_all:
        return np.zeros((n, 0)), np.zeros((n, 0))
    return np.concatenate(th_all, 1), np.concatenate(rate_all, 1)


def place_target(sys, dqp, qp, idx, env_ids, field, episode, seed):
    """Marker placement (R36): pos[idx, T] = x̄_T + range ⊙ u(env, T, field, episode)."""
    g = sys.task.goal
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    key = (seed & 0xFFFFFFFF, seed >> 32)
    for i, e, f, k in zip(idx, env_ids, field, episode):
        x = philox4x32_10((int(e), g.target, int(f), int(k)), key)
        for c in range(3):
            qp["pos"][i, g.target, c] = dqp["pos"][g.target, c] + g.range[c] * uniform_pm1(x[c])


class Env:
    """An Oracle whose scene has a `task` block."""

    def __init__(self, oracle):
        if oracle.sys.task is None:
            raise ValueError("scene has no task block")
        self.o = oracle
        self.sys = oracle.sys
        self.task = oracle.sys.task

    @property
    def obs_dim(self):
        return self.sys.obs_dim

    def observe(self, qp, contact_dv=None):
        t, s = self.task, self.sys
        n = qp["pos"].shape[0]
        th, rate = joint_angles_and_rates(s, qp)
        parts = [qp["pos"][:, t.torso, 2:3], qp["rot"][:, t.torso], th,
                 qp["vel"][:, t.torso], qp["ang"][:, t.torso], rate]
        if t.goal is not None:
            xo, xt = qp["pos"][:, t.goal.obj], qp["pos"][:, t.goal.target]
            parts += [xt - xo, xo - qp["pos"][:, t.torso], qp["vel"][:, t.goal.obj]]
        if t.contact_obs:
            cdv = np.zeros((n, len(s.bodies), 6)) if contact_dv is None else contact_dv
            parts.append(np.clip(cdv, -1.0, 1.0).reshape(n, -1))
        obs = np.concatenate([np.asarray(p, dtype=np.float64).reshape(n, -1) for p in parts], 1)
        assert obs.shape == (n, self.obs_dim)
        return obs

    def reset(self, n, seed, env_offset=0):
        """brax_env_reset: episode-0 reset noise, steps = episode = 0, obs."""
        t = self.task
        dqp = self.o.default_qp()
        qp = reset_qp(self.sys, dqp, n, seed, t.reset_vel_noise, t.reset_ang_noise, env_ids=env_offset + np.arange(n))
        if t.goal is not None:
            place_target(self.sys, dqp, qp, range(n), env_offset + np.arange(n), [2] * n, [0] * n, seed)
        steps = np.zeros(n, dtype=np.int32)
        episode = np.zeros(n, dtype=np.uint32)
        return qp, steps, episode, self.observe(qp)

    def step(self, qp, steps, episode, action, seed, env_offset=0, threads=1):
        t, s = self.task, self.sys
        n = qp["pos"].shape[0]
        g = t.goal
        ob = t.torso if g is None else g.obj
        x0 = np.asarray(qp["pos"][:, ob], dtype=np.float64).copy()
        q1, ex = self.o.step(qp, action, threads=threads, contact_dv=t.contact_obs)
        x1 = q1["pos"][:, ob].copy()
        a = np.zeros((n, 0)) if action is None else np.asarray(action, dtype=np.float64).reshape(n, -1)
        steps1 = np.asarray(steps, dtype=np.int64) + 1
        d1 = None
        if g is None:
            reward = ((x1 - x0) @ t.forward) / s.dt
        else:  # R36: progress towards the marker, which the frozen body keeps in place during the step
            xt = np.asarray(q1["pos"][:, g.target], dtype=np.float64)
            d0 = np.linalg.norm(x0 - xt, axis=1)
            d1 = np.linalg.norm(x1 - xt, axis=1)
            hit = d1 < g.radius
            reward = (d0 - d1) / s.dt + g.bonus * hit
            if hit.any():
                idx = np.nonzero(hit)[0]
                place_target(s, self.o.default_qp(), q1, idx, env_offset + idx, 2 + steps1[idx],
                             np.asarray(episode, dtype=np.int64)[idx], seed)
        reward = reward + t.survive_reward - t.ctrl_cost * np.sum(a * a, 1)
        done = steps1 >= t.episode_length
        xz = q1["pos"][:, t.torso, 2].copy()
        if t.healthy_z is not None:
            z = xz
            done = done | (z < t.healthy_z[0]) | (z > t.healthy_z[1])
        episode1 = np.asarray(episode, dtype=np.int64) + done
        steps1 = np.where(done, 0, steps1)
        cdv = ex.get("contact_dv")
        if done.any():
            idx = np.nonzero(done)[0]
            dqp = self.o.default_qp()
            r = reset_qp(s, dqp, len(idx), seed, t.reset_vel_noise, t.reset_ang_noise,
                         env_ids=env_offset + idx, episode=episode1[idx])
            if g is not None:
                place_target(s, dqp, r, range(len(idx)), env_offset + idx, [2] * len(idx), episode1[idx], seed)
            for k in q1:
                q1[k][idx] = r[k]
            if cdv is not None:
                cdv[idx] = 0.0
        return {"qp": q1, "obs": self.observe(q1, cdv), "reward": reward, "done": done,
                "steps": steps1.astype(np.int32), "episode": episode1.astype(np.uint32),
                "ambiguous": ex["ambiguous"], "status": ex["status"], "x1_z": xz, "d1": d1}
