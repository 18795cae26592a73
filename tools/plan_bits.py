"""Diagnostic: does an env's result depend on the launch plan?  Steps the same
states under plan (1,1) and each other plan and reports the fields / envs that
differ bitwise (scenes at their own substeps and at substeps 1).
    python tools/plan_bits.py [--scenes ball,pendulum,chain2,coverage,ant]"""
import argparse
import os
import re
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--scenes", default="ball,pendulum,chain2,coverage,ant,humanoid")
p.add_argument("--envs", type=int, default=256)
a = p.parse_args()
FIELDS = ("pos", "rot", "vel", "ang")
for name in a.scenes.split(","):
    with open(os.path.join(ROOT, "scenes", f"{name}.bxc")) as f:
        text = f.read()
    for sub in (None, 1):
        t = text if sub is None else re.sub(r"^substeps: *\d+", "substeps: 1", text, flags=re.M)
        s = bx.System(t)
        qp0 = s.alloc_qp(a.envs)
        s.reset(qp0, seed=3, vel_noise=0.5, ang_noise=0.5)
        act = torch.from_numpy(synth.actions(5, 1, a.envs, s.act_dim)[0]).cuda() if s.act_dim else None
        res = {}
        for plan in ("1,1", "2,1", "1,2", "2,2", "4,2"):
            os.environ["BRAX_PLAN"] = plan
            out = s.alloc_qp(a.envs)
            s.step(qp0, act, out)
            torch.cuda.synchronize()
            res[plan] = {k: out[k].cpu().numpy() for k in FIELDS}
        os.environ.pop("BRAX_PLAN")
        for plan in res:
            if plan == "1,1":
                continue
            diffs = []
            for k in FIELDS:
                d = res[plan][k] != res["1,1"][k]
                if d.any():
                    envs = np.nonzero(d.reshape(a.envs, -1).any(1))[0]
                    mx = np.max(np.abs(res[plan][k] - res["1,1"][k]))
                    diffs.append(f"{k}: {len(envs)} envs (first {envs[:4].tolist()}), max {mx:.2e}")
            print(f"{name:10s} substeps={'own' if sub is None else 1} plan {plan}: " + ("; ".join(diffs) if diffs else "bitwise equal"))
