"""Measured spread of brax_step_jvp vs the oracle's central differences."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import test_gpu_jvp as T  # noqa: E402
from oracle.diff import jvp_fd  # noqa: E402
import paper_2106_13281_b200 as bx  # noqa: E402

for name in ["pendulum", "chain2", "ball", "ant", "humanoid", "halfcheetah", "grasp", "fetch", "coverage"]:
    text = oracle.load_scene(name)
    o, s = oracle.Oracle(text), bx.System(text)
    n = 200
    qp = T.states(o, n, seed=3, T0=5)
    act = synth.actions(4, 1, n, o.act_dim)[0] if o.act_dim else None
    dq, da = T.tangents(o, n, seed=5)
    ref, kink = jvp_fd(o, qp, act, dq, da, threads=8)
    a_t = torch.from_numpy(act).cuda() if o.act_dim else None
    out, dout = s.step_jvp(T.dev(qp), a_t, T.dev(dq), torch.from_numpy(da.astype(np.float32)).cuda() if o.act_dim else None)
    got = T.host(dout)
    worst = 0.0
    for k in T.FIELDS:
        err = np.abs(got[k] - ref[k]).reshape(n, -1).max(1)
        scale = 1.0 + np.abs(ref[k]).reshape(n, -1).max(1)
        worst = max(worst, float((err / scale)[~kink].max()))
    print(f"{name:12s} kink {kink.sum():3d}/{n}  max rel err {worst:.2e}")
