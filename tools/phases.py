"""Per-phase cycle breakdown of the step kernel (brax_system_set_tracing).
    python tools/phases.py [--scenes ant] [--envs 8192]"""
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
p.add_argument("--scenes", default="ant")
p.add_argument("--envs", default="2048,8192,65536")
p.add_argument("--steps", type=int, default=50)
p.add_argument("--plans", default="", help="comma-separated 'G:V' launch plans (default: the library's choice)")
a = p.parse_args()
for scene in a.scenes.split(","):
    s = bx.System(open(os.path.join(ROOT, "scenes", f"{scene}.bxc")).read())
    for n, plan in [(int(x), pl) for x in a.envs.split(",") for pl in (a.plans.split(",") if a.plans else [""])]:
        if plan:
            os.environ["BRAX_PLAN"] = plan.replace(":", ",")
        else:
            os.environ.pop("BRAX_PLAN", None)
        qp = s.alloc_qp(n)
        s.reset(qp, 0, 0.1, 0.1)
        acts = torch.from_numpy(synth.actions(1, a.steps, n, s.act_dim)).cuda() if s.act_dim else None
        for t in range(5):
            s.step(qp, acts[t] if acts is not None else None, qp)
        torch.cuda.synchronize()
        s.set_tracing(True)
        s.phase_cycles()
        for t in range(a.steps):
            s.step(qp, acts[t] if acts is not None else None, qp)
        torch.cuda.synchronize()
        cyc = s.phase_cycles()
        s.set_tracing(False)
        cfg = s.launch_config(n)
        blocks = (n + cfg["E"] - 1) // cfg["E"]
        per = [c / (a.steps * blocks) for c in cyc]
        tot = sum(per)
        print(json.dumps({"scene": scene, "envs": n, "plan": [cfg["G"], cfg["V"]], "cycles_per_block_step": [round(x) for x in per],
                          "share": [round(x / tot, 3) for x in per],
                          "per_substep_B_C": [round(per[1] / s.substeps), round(per[2] / s.substeps)]}))
