"""Diagnostic for the 100-step parity bar: GPU vs oracle over a
free-running 100-step trajectory, per-env max error, and the excluded envs
under the standard R23 band (1e-5) and the widened one (1e-4).

    python tools/parity100.py [--scene ant] [--n 512] [--T 100] [--zero]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

FIELDS = ("pos", "rot", "vel", "ang")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--scene", default="ant")
    p.add_argument("--n", type=int, default=512)
    p.add_argument("--T", type=int, default=100)
    p.add_argument("--zero", action="store_true")
    p.add_argument("--seed", type=int, default=11)
    a = p.parse_args()
    text = oracle.load_scene(a.scene)
    o = oracle.Oracle(text)
    s = bx.System(text)
    n, T = a.n, a.T
    qp = synth.to_f32(o.reset(n, a.seed, 0.1, 0.1))
    acts = synth.actions(a.seed + 1, T, n, o.act_dim)
    if a.zero:
        acts[:] = 0
    bands = {"r23": 1e-5, "wide": 1e-4}
    amb = {}
    ref = None
    for name, b in bands.items():
        ob = oracle.Oracle(o.sys, amb_d=b, amb_jn=b)
        r, info = ob.rollout({k: v.astype(np.float64) for k, v in qp.items()}, acts, threads=os.cpu_count())
        amb[name] = info["ambiguous"] if info["ambiguous"] is not None else np.zeros(n, bool)
        ref = r
    qd = {k: torch.from_numpy(qp[k]).cuda() for k in FIELDS}
    ad = torch.from_numpy(acts).cuda() if o.act_dim else None
    for t in range(T):
        s.step(qd, ad[t] if ad is not None else None, qd)
    torch.cuda.synchronize()
    got = {k: qd[k].cpu().numpy().astype(np.float64) for k in FIELDS}
    per_env = np.max(np.stack([np.abs(got[k] - ref[k]).reshape(n, -1).max(1) for k in FIELDS]), axis=0)
    out = {"scene": a.scene, "n": n, "T": T, "zero_action": a.zero}
    for name in bands:
        keep = ~amb[name]
        out[name] = {"excluded": int((~keep).sum()), "max_err_kept": float(per_env[keep].max()) if keep.any() else 0,
                     "kept_over_1e-3": int((per_env[keep] > 1e-3).sum())}
    out["err_quantiles_all"] = [float(x) for x in np.quantile(per_env, [0.5, 0.9, 0.99, 1.0])]
    out["over_1e-3_all"] = int((per_env > 1e-3).sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
