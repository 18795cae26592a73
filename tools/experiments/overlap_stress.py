"""Stress of the launch overlap: long in-place chains (graphs and eager) at several batch
sizes / scenes against the same launches serialised; prints mismatches (expect none)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

bad = 0
for scene, n, T in (("ant", 8192, 400), ("ant", 65536, 60), ("ant", 777, 300), ("humanoid", 4096, 300),
                    ("fetch", 2048, 300), ("halfcheetah", 3000, 300)):
    o = oracle.Oracle(oracle.load_scene(scene))
    s = bx.System(oracle.load_scene(scene))
    q0 = {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).cuda() for k, v in o.reset(n, 3, 0.1, 0.1).items()}
    acts = torch.from_numpy(synth.actions(4, 16, n, o.act_dim)).cuda()
    s.tune(q0, acts[0])
    X = {k: v.clone() for k, v in q0.items()}
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=st):
        for t in range(T):
            s.step(X, acts[t % 16], X)
    for k in X:
        X[k].copy_(q0[k])
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    E = {k: v.clone() for k, v in q0.items()}
    for t in range(T):
        s.step(E, acts[t % 16], E)
    torch.cuda.synchronize()
    R = {k: v.clone() for k, v in q0.items()}
    for t in range(T):
        s.step(R, acts[t % 16], R)
        torch.cuda.synchronize()
    for name, Y in (("graph", X), ("eager", E)):
        for k in R:
            if not torch.equal(Y[k], R[k]):
                bad += 1
                print("MISMATCH", scene, n, name, k, flush=True)
    print("ok" if bad == 0 else "bad", scene, n, T, flush=True)
print("mismatches", bad)
