"""Cost of the NEXT-1 env epilogue (ant, 8192 envs, CUDA graph over 23 rotating
batches): physics-only brax_step vs brax_env_step without and with observations."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

n, R = int(os.environ.get("N", 8192)), 23
s = bx.System(open(os.path.join(ROOT, "scenes", "ant.bxc")).read())
od = s.task_info()["obs_dim"]
sets, acts, est = [], [], []
for r in range(R):
    q = s.alloc_qp(n)
    s.reset(q, r, 0.1, 0.1)
    sets.append(q)
    acts.append(torch.from_numpy(synth.actions(r, 1, n, s.act_dim)[0]).cuda())
    est.append({"steps": torch.zeros(n, dtype=torch.int32, device="cuda"),
                "episode": torch.zeros(n, dtype=torch.int32, device="cuda"),
                "obs": torch.empty((n, od), device="cuda"), "reward": torch.empty(n, device="cuda"),
                "done": torch.empty(n, dtype=torch.uint8, device="cuda")})
s.tune(sets[0], acts[0])
res = {"cfg": s.launch_config(n)}


def run(kind):
    for r in range(R):
        if kind == "physics":
            s.step(sets[r], acts[r], sets[r])
        else:
            st = est[r]
            bx.brax_env_step(s.handle, sets[r], acts[r], 1, sets[r], n, st["obs"] if kind == "env_obs" else None,
                             st["reward"], st["done"], st["steps"], st["episode"], seed=1)


for kind in ("physics", "env_noobs", "env_obs"):
    for _ in range(2):
        run(kind)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run(kind)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        g.replay()
    e1.record()
    e1.synchronize()
    res[kind + "_us"] = e0.elapsed_time(e1) * 1e3 / (10 * R)
print(json.dumps(res))
