"""NEXT-3: the "astronaut" conservation diagnostic of Fig. 5 (PAPER.md:251-258,
:264), run on the GPU step kernel.

Protocol (paper, after Erez et al.): the humanoid with damping, collisions and
gravity disabled; (momentum) limbs randomly actuated for 1 s with ≈ 0.5 N·m
per actuator per step; (energy) actuators disabled, every body part given a
random 1 m/s kick, energy drift measured after 1 s; averaged over 128 seeds,
single precision.  Fidelity axis: the substep length h (dt fixed, substeps
2, 4, 8, 16; at 1 substep the undamped humanoid's stiff springs are beyond the
explicit scheme's stability limit, R6).

Quantities (host-side analysis of the GPU's QP, fp64):
  P = Σ m v;  L = Σ (x × m v + I_w ω) about the origin (isotropic inertia, R4);
  E = Σ ½ m|v|² + ½ ω·I_w ω + Σ_joints [½ k |Δx|² + ½ k_a Σ_{i≥d} θ_i²
      + ½ k_l Σ_{i<d} (θ_i − clamp(θ_i, lo_i, hi_i))²]  (anchor, alignment and limit
      springs; θ the joint's intrinsic X-Y-Z angles, R7).
    python tools/astronaut.py [--seeds 128] [--json out.json]
"""
from __future__ import annotations

import argparse
import json
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def astronaut_text(substeps: int, strength: float, dt: float | None = None) -> str:
    """humanoid.bxc with gravity, damping and colliders removed, torque actuators of `strength`
    (and the step length dt, if given)."""
    with open(os.path.join(ROOT, "scenes", "humanoid.bxc")) as f:
        t = f.read()
    if dt is not None:
        t = re.sub(r"^dt: *[0-9.]+", f"dt: {dt}", t, flags=re.M)
    t = re.sub(r"gravity \{[^}]*\}", "gravity { }", t)
    t = re.sub(r"angular_damping: [0-9.]+", "angular_damping: 0", t)
    t = re.sub(r"\n  colliders \{[^\n]*\} \}", " }", t)       # each body's one-line collider block
    t = re.sub(r"collide_include \{[^}]*\}\n", "", t)
    t = re.sub(r'bodies \{ name: "Ground" frozen \{ all: true \} colliders \{ plane \{\} \} \}\n', "", t)
    t = re.sub(r"strength: [0-9.]+", f"strength: {strength}", t)
    t = re.sub(r"^substeps: *\d+", f"substeps: {substeps}", t, flags=re.M)
    assert "colliders" not in t and "collide_include" not in t
    return t


def quat_rotate(q, v):
    w, u = q[..., :1], q[..., 1:]
    t = 2.0 * np.cross(u, v)
    return v + w * t + np.cross(u, t)


def invariants(o_sys, qp):
    """P, L (about the origin) and total mechanical energy per env (fp64)."""
    m = np.array([b.mass for b in o_sys.bodies])[None, :, None]
    I = np.array([b.inertia for b in o_sys.bodies])[None]
    x, q, v, w = (qp[k].astype(np.float64) for k in ("pos", "rot", "vel", "ang"))
    P = (m * v).sum(1)
    # I_w ω = R (I ⊙ Rᵀ ω)
    wb = quat_rotate(q * np.array([1, -1, -1, -1]), w)
    Iw = quat_rotate(q, I * wb)
    L = (np.cross(x, m * v) + Iw).sum(1)
    ke = 0.5 * (m[..., 0] * (v * v).sum(-1)).sum(1) + 0.5 * (w * Iw).sum(-1).sum(1)
    pe = np.zeros(x.shape[0])
    for j in o_sys.joints:
        ap = x[:, j.parent] + quat_rotate(q[:, j.parent], j.parent_offset)
        ac = x[:, j.child] + quat_rotate(q[:, j.child], j.child_offset)
        pe += 0.5 * j.stiffness * ((ap - ac) ** 2).sum(-1)
        th = joint_angles(q[:, j.parent], q[:, j.child], j)
        for i in range(3):
            if i < j.dof:
                excess = th[:, i] - np.clip(th[:, i], j.limits[i, 0], j.limits[i, 1])
                pe += 0.5 * j.limit_stiffness * excess ** 2
            else:
                pe += 0.5 * j.angular_stiffness * th[:, i] ** 2
    return P, L, ke + pe


def qmul(a, b):
    aw, ax, ay, az = np.moveaxis(a, -1, 0)
    bw, bx, by, bz = np.moveaxis(b, -1, 0)
    return np.stack([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw], -1)


def joint_angles(qp, qc, j):
    """Intrinsic X-Y-Z angles of conj(q_p⊗J_p)⊗(q_c⊗J_c) (analysis copy of R7's extraction)."""
    conj = np.array([1, -1, -1, -1])
    jc = qmul(j.reference_rotation * conj, j.rotation)
    qr = qmul(qmul(qp, np.broadcast_to(j.rotation, qp.shape)) * conj, qmul(qc, np.broadcast_to(jc, qc.shape)))
    qr = np.where(qr[:, :1] < 0, -qr, qr)
    w, x, y, z = qr.T
    return np.stack([np.arctan2(-2 * (y * z - w * x), 1 - 2 * (x * x + y * y)),
                     np.arcsin(np.clip(2 * (x * z + w * y), -1, 1)),
                     np.arctan2(-2 * (x * y - w * z), 1 - 2 * (y * y + z * z))], -1)


def run(seeds=128, substeps_list=(2, 4, 8, 16), horizon_s=1.0):
    import torch

    import oracle
    import paper_2106_13281_b200 as bx
    import synth
    out = []
    for S in substeps_list:
        text_mom = astronaut_text(S, 0.5)
        text_en = astronaut_text(S, 0.0)
        sys_m = bx.System(text_mom)
        sys_e = bx.System(text_en)
        o = oracle.parse_system(text_mom)  # host-side constants for the analysis only
        dt = o.dt
        steps = int(round(horizon_s / dt))
        # momentum: random ±0.5 N·m torques every step
        qp = sys_m.alloc_qp(seeds)
        sys_m.reset(qp, seed=S, vel_noise=0.1, ang_noise=0.1)
        acts = torch.from_numpy(synth.actions(100 + S, steps, seeds, sys_m.act_dim)).cuda()
        q0 = {k: v.cpu().numpy() for k, v in qp.items()}
        for t in range(steps):
            sys_m.step(qp, acts[t], qp)
        torch.cuda.synchronize()
        q1 = {k: v.cpu().numpy() for k, v in qp.items()}
        P0, L0, _ = invariants(o, q0)
        P1, L1, _ = invariants(o, q1)
        # energy: no actuation, 1 m/s random kick of every body (random unit directions)
        qe = sys_e.alloc_qp(seeds)
        sys_e.reset(qe, seed=S, vel_noise=0.0, ang_noise=0.0)
        rng = np.random.Generator(np.random.PCG64(200 + S))
        kick = rng.normal(size=qe["vel"].shape)
        kick /= np.linalg.norm(kick, axis=-1, keepdims=True)
        qe["vel"].copy_(torch.from_numpy(kick.astype(np.float32)))
        e0 = {k: v.cpu().numpy() for k, v in qe.items()}
        zero = torch.zeros((steps, seeds, sys_e.act_dim), device="cuda")
        for t in range(steps):
            sys_e.step(qe, zero[t], qe)
        torch.cuda.synchronize()
        e1 = {k: v.cpu().numpy() for k, v in qe.items()}
        _, _, E0 = invariants(o, e0)
        _, _, E1 = invariants(o, e1)
        out.append({"substeps": S, "h": dt / S, "steps": steps, "seeds": seeds,
                    "linear_momentum_drift": float(np.mean(np.linalg.norm(P1 - P0, axis=-1))),
                    "angular_momentum_drift": float(np.mean(np.linalg.norm(L1 - L0, axis=-1))),
                    "energy_drift": float(np.mean(np.abs(E1 - E0))),
                    "energy_rel_drift": float(np.mean(np.abs(E1 - E0) / np.abs(E0)))})
    return out


def run_dt_ladder(seeds=16, dts=(0.02, 0.01, 0.005, 0.0025), substeps=4, horizon_s=1.0, engine="gpu"):
    """The Fig. 5 fidelity axis (steps per second): the same two protocols
    at a ladder of step lengths dt (substeps fixed), on the GPU kernel or on the fp64 oracle,
    from identical inputs (brax_reset's Philox noise = oracle.reset; the same NumPy actions and
    kicks).  Returns one dict per dt with mean drifts over the seeds and the per-seed energy
    drift."""
    import oracle
    import synth
    out = []
    for dt in dts:
        text_mom, text_en = astronaut_text(substeps, 0.5, dt), astronaut_text(substeps, 0.0, dt)
        o_m, o_e = oracle.Oracle(text_mom), oracle.Oracle(text_en)
        steps = int(round(horizon_s / dt))
        acts = synth.actions(300 + int(1e4 * dt), steps, seeds, o_m.act_dim)
        q0 = o_m.reset(seeds, 7, 0.1, 0.1)
        e0 = o_e.reset(seeds, 7, 0.0, 0.0)
        rng = np.random.Generator(np.random.PCG64(400 + int(1e4 * dt)))
        kick = rng.normal(size=e0["vel"].shape)
        kick /= np.linalg.norm(kick, axis=-1, keepdims=True)
        e0["vel"] = kick
        q0 = synth.to_f32(q0)
        e0 = synth.to_f32(e0)
        if engine == "oracle":
            q1, _ = o_m.rollout(q0, acts, threads=8)
            e1, _ = o_e.rollout(e0, np.zeros((steps, seeds, o_e.act_dim), np.float32), threads=8)
        else:
            import torch

            import paper_2106_13281_b200 as bx
            sys_m, sys_e = bx.System(text_mom), bx.System(text_en)
            qd = {k: torch.from_numpy(v).cuda() for k, v in q0.items()}
            ed = {k: torch.from_numpy(v).cuda() for k, v in e0.items()}
            ad = torch.from_numpy(acts).cuda()
            zero = torch.zeros((seeds, sys_e.act_dim), device="cuda")
            for t in range(steps):
                sys_m.step(qd, ad[t], qd)
                sys_e.step(ed, zero, ed)
            torch.cuda.synchronize()
            q1 = {k: v.cpu().numpy() for k, v in qd.items()}
            e1 = {k: v.cpu().numpy() for k, v in ed.items()}
        P0, L0, _ = invariants(o_m.sys, q0)
        P1, L1, _ = invariants(o_m.sys, q1)
        _, _, E0 = invariants(o_e.sys, e0)
        _, _, E1 = invariants(o_e.sys, e1)
        out.append({"engine": engine, "dt": dt, "substeps": substeps, "steps": steps, "seeds": seeds,
                    "linear_momentum_drift": float(np.mean(np.linalg.norm(P1 - P0, axis=-1))),
                    "angular_momentum_drift": float(np.mean(np.linalg.norm(L1 - L0, axis=-1))),
                    "energy_drift": float(np.mean(np.abs(E1 - E0))),
                    "energy_rel_drift": float(np.mean(np.abs(E1 - E0) / np.abs(E0))),
                    "energy_drift_per_seed": (E1 - E0).tolist(), "energy0_per_seed": E0.tolist()})
    return out


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("--seeds", type=int, default=128)
    p.add_argument("--json", default=None)
    p.add_argument("--dt-ladder", action="store_true", help="GPU and oracle over dt in {0.02, 0.01, 0.005, 0.0025}")
    a = p.parse_args()
    if a.dt_ladder:
        res = []
        for eng in ("oracle", "gpu"):
            res += run_dt_ladder(min(a.seeds, 16), engine=eng)
        for r in res:
            r.pop("energy_drift_per_seed")
            r.pop("energy0_per_seed")
    else:
        res = run(a.seeds)
    for r in res:
        print(json.dumps(r))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)
