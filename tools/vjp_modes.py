"""brax_step_vjp with the hand-derived joint adjoint vs all item adjoints from local
value+tangent evaluations (BRAX_VJP_LOCAL_AD=1), 8192 envs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2106_13281_b200 as bx, synth
for scene in ("ant", "humanoid"):
    s = bx.System(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scenes", f"{scene}.bxc")).read())
    n = 8192
    qp = s.alloc_qp(n); s.reset(qp, 0, 0.1, 0.1)
    act = torch.from_numpy(synth.actions(1, 1, n, s.act_dim)[0]).cuda()
    g = {k: torch.randn_like(v) for k, v in qp.items()}
    res = {}
    for mode in ("0", "1"):
        if mode == "1":
            os.environ["BRAX_VJP_LOCAL_AD"] = "1"
        else:
            os.environ.pop("BRAX_VJP_LOCAL_AD", None)
        s.step_vjp(qp, act, g); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): s.step_vjp(qp, act, g)
        e1.record(); torch.cuda.synchronize()
        res[{"0": "hand_joint", "1": "local_ad"}[mode]] = e0.elapsed_time(e1) / 5 * 1e3
    print(scene, json.dumps(res))
