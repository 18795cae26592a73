"""Algorithmic flop / MUFU / byte counts per env-step for each benchmark scene
(SURVEY.md §8(d) counting convention), from the oracle's op-counting scalar
run along seeded random-action trajectories (the bench workload's recipe:
reset with vel/ang noise 0.1, then U(−1, 1) actions).

Writes profiles/algorithmic_counts.json, which bench.py reads for the
roofline's `achieved` (bench.py itself never runs the oracle outside its
cpu_baseline leg).  Calls only oracle/ and synth.

    python tools/count_flops.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402

SCENES = ["ball", "pendulum", "chain2", "ant", "humanoid", "halfcheetah", "grasp", "fetch", "coverage"]


def count(name, n=64, burn=30, measure=20, seed=0):
    o = oracle.Oracle(oracle.load_scene(name))
    qp = o.reset(n, seed, 0.1, 0.1)
    acts = synth.actions(seed + 1, burn + measure, n, o.act_dim)
    fl = mu = fl_lean = mu_lean = 0
    active = 0.0
    for t in range(burn + measure):
        if t >= burn:
            f, m = o.count_ops(qp, acts[t])
            fl += f
            mu += m
            f, m = o.count_ops(qp, acts[t], lean=True)
            fl_lean += f
            mu_lean += m
        qp, ex = o.step(qp, acts[t], threads=8)
        if t >= burn and o.n_slots:
            active += ex["contact_active"].sum() / (o.sys.substeps * n)
    steps = n * measure
    B, A = o.n_bodies, o.act_dim
    return {
        "flops_per_env_step": fl / steps,
        "mufu_per_env_step": mu / steps,
        "flops_per_env_step_lean": fl_lean / steps,
        "mufu_per_env_step_lean": mu_lean / steps,
        "bytes_per_env_step": 4 * (26 * B + A),
        "active_contacts_per_substep": active / measure,
        "n_bodies": B, "act_dim": A, "n_slots": o.n_slots, "substeps": o.sys.substeps,
        "sample": f"{n} envs, steps {burn}..{burn + measure - 1} of a seeded random-action rollout",
    }


if __name__ == "__main__":
    out = {"convention": "add/sub/mul 1 flop, div/sqrt 4 flops + 1 MUFU, atan2/asin 20 flops + 1 MUFU "
                         "(SURVEY.md §8(d)); bytes = full QP read + write + action read = 4*(26*B + A); "
                         "*_lean: the same with the operations an exactly neutral scene value makes (unit "
                         "masks, isotropic inertia, zero damping, zero collider offset, identity collider "
                         "rotation) not counted",
           "scenes": {}}
    for s in SCENES:
        out["scenes"][s] = count(s)
        print(s, {k: round(v, 1) if isinstance(v, float) else v for k, v in out["scenes"][s].items()})
    with open(os.path.join(ROOT, "profiles", "algorithmic_counts.json"), "w") as f:
        json.dump(out, f, indent=1)
