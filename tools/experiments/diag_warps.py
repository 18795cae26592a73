"""Per-warp clock stamps of one substep (build with BRAX_NVCC_FLAGS=-DBRAX_DIAG):
phase-1 work, wait at the mid barrier, phase-2 work.
    BRAX_DIAG_BLOCK=1 BRAX_PLAN=2,2 python tools/experiments/diag_warps.py [n_envs] [scene | path.bxc]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
scene = sys.argv[2] if len(sys.argv) > 2 else "ant"
path = scene if scene.endswith(".bxc") else os.path.join(ROOT, "scenes", f"{scene}.bxc")
s = bx.System(open(path).read())
qp = s.alloc_qp(n)
s.reset(qp, 0, 0.1, 0.1)
acts = torch.from_numpy(synth.actions(1, 20, n, s.act_dim)).cuda()
for t in range(20):
    s.step(qp, acts[t], qp)
torch.cuda.synchronize()
print("cfg", s.launch_config(n), flush=True)
