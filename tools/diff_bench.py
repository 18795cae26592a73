"""Cost of the NEXT-4 derivative calls vs the plain step (ant, 8192 envs).
    python tools/diff_bench.py [--scene ant] [--envs 8192]"""
import argparse
import json
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
a = p.parse_args()
s = bx.System(open(os.path.join(ROOT, "scenes", f"{a.scene}.bxc")).read())
n = a.envs
qp = s.alloc_qp(n)
s.reset(qp, 0, 0.1, 0.1)
act = torch.from_numpy(synth.actions(1, 1, n, s.act_dim)[0]).cuda()
dq = {k: torch.randn_like(v) * 1e-3 for k, v in qp.items()}
out = s.alloc_qp(n)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # µs


t_step = timed(lambda: s.step(qp, act, out), 200)
t_jvp = timed(lambda: s.step_jvp(qp, act, dq), 50)
t_vjp = timed(lambda: s.step_vjp(qp, act, dq), 10)
os.environ["BRAX_VJP_COLUMNS"] = "1"
t_cols = timed(lambda: s.step_vjp(qp, act, dq), 3)
os.environ.pop("BRAX_VJP_COLUMNS")
print(json.dumps({"scene": a.scene, "envs": n, "step_us": t_step, "jvp_us": t_jvp, "vjp_us": t_vjp,
                  "vjp_columns_us": t_cols, "jvp_over_step": t_jvp / t_step, "vjp_over_step": t_vjp / t_step,
                  "vjp_columns_over_step": t_cols / t_step, "vjp_launches": 1,
                  "vjp_columns_launches": 3 * (13 * s.n_bodies + s.act_dim)}))
