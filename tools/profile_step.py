"""Minimal workload for ncu: ant (or --scene), N envs, a few brax_step launches.

    python tools/profile_step.py [--scene ant] [--envs 8192] [--steps 6]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--scene", default="ant")
p.add_argument("--envs", type=int, default=8192)
p.add_argument("--steps", type=int, default=6)
p.add_argument("--rollout", type=int, default=0, help="also run one brax_rollout of this many steps")
a = p.parse_args()
with open(os.path.join(ROOT, "scenes", f"{a.scene}.bxc")) as f:
    s = bx.System(f.read())
qp = s.alloc_qp(a.envs)
s.reset(qp, seed=0, vel_noise=0.1, ang_noise=0.1)
acts = torch.from_numpy(synth.actions(1, max(a.steps, a.rollout, 1), a.envs, s.act_dim)).cuda() if s.act_dim else None
for t in range(a.steps):
    s.step(qp, acts[t] if acts is not None else None, qp)
if a.rollout:
    s.rollout(qp, acts[: a.rollout], qp)
torch.cuda.synchronize()
print("ok", a.scene, a.envs, float(qp["pos"][:, 1, 2].mean()))
