import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import oracle, synth
from oracle.env import Env
import paper_2106_13281_b200 as bx
import test_gpu_env as T
for name in T.ENV_SCENES:
    e, s = T.scene(name)
    n = 1000
    qp, steps, ep = T.start_states(e, n, seed=31)
    act = synth.actions(32, 1, n, e.sys.act_dim)[0]
    ref = e.step(qp, steps, ep, act, seed=9, env_offset=50, threads=8)
    st = {"qp": {k: T.dev(qp[k]) for k in T.FIELDS}, "steps": T.dev(steps, torch.int32), "episode": T.dev(ep.view(np.int32), torch.int32)}
    out = s.env_step(st, T.dev(act), seed=9, env_offset=50)
    keep = ~ref["ambiguous"] & ~T.near_threshold(e, ref["x1_z"])
    r = out["reward"][0].cpu().numpy(); o = out["obs"][0].cpu().numpy()
    err_o = np.abs(o[keep] - ref["obs"][keep]).max(0)
    print(name, "keep", keep.sum(), "done", ref["done"].sum(), "reward err", np.abs(r[keep]-ref["reward"][keep]).max(), "obs err max", err_o.max(), "argmax col", err_o.argmax(), "qp err", max(np.abs(st["qp"][k].cpu().numpy()[keep]-ref["qp"][k][keep]).max() for k in T.FIELDS))
