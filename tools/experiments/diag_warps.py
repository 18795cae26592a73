"""Per-warp clock stamps of one substep (BRAX_DIAG_BLOCK): phase-1 work, wait at the
mid barrier, phase-2 work (+ wait at the next barrier is the remainder).
    BRAX_DIAG_BLOCK=1 BRAX_PLAN=2,2 python tools/experiments/diag_warps.py [n_envs] [scene]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
scene = sys.argv[2] if len(sys.argv) > 2 else "ant"
s = bx.System(open(os.path.join(ROOT, "scenes", f"{scene}.bxc")).read())
qp = s.alloc_qp(n)
s.reset(qp, 0, 0.1, 0.1)
acts = torch.from_numpy(synth.actions(1, 20, n, s.act_dim)).cuda()
for t in range(20):
    s.step(qp, acts[t], qp)
torch.cuda.synchronize()
print("cfg", s.launch_config(n), flush=True)
