"""Specialised vs generic kernel on the GPU: bitwise/ULP agreement and speed."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

for scene in sys.argv[1:] or ["ant", "humanoid", "halfcheetah", "grasp", "fetch", "pendulum", "ball"]:
    text = open(os.path.join(ROOT, "scenes", f"{scene}.bxc")).read()
    os.environ["BRAX_SPECIALIZE"] = "0"
    gen = bx.System(text)
    os.environ["BRAX_SPECIALIZE"] = "1"
    spec = bx.System(text)
    print(scene, "specialized:", spec.info.specialized, spec.kernel_log().strip().replace("\n", " | ")[-300:])
    n = 8192
    qa = gen.alloc_qp(n)
    gen.reset(qa, 0, 0.1, 0.1)
    qb = {k: v.clone() for k, v in qa.items()}
    acts = torch.from_numpy(synth.actions(1, 20, n, gen.act_dim)).cuda() if gen.act_dim else None
    for t in range(20):
        gen.step(qa, acts[t] if acts is not None else None, qa)
        spec.step(qb, acts[t] if acts is not None else None, qb)
    torch.cuda.synchronize()
    d = max(float((qa[k] - qb[k]).abs().max()) for k in qa)
    print(f"  max |generic - specialized| after 20 steps: {d:.3g}")
    for name, s in (("generic", gen), ("specialized", spec)):
        q = {k: v.clone() for k, v in qa.items()}
        for _ in range(3):
            s.step(q, acts[0] if acts is not None else None, q)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for t in range(100):
            s.step(q, acts[t % 20] if acts is not None else None, q)
        e1.record()
        torch.cuda.synchronize()
        print(f"  {name:12s} {e0.elapsed_time(e1) * 10:.1f} us/step at {n} envs")
