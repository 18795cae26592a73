"""End-to-end pipelining study (ant, 8192 envs): pinned host qp+actions -> device ->
brax_step -> host, per step.  Variants: NS streams round-robin (bench's scheme), and
a three-stage pipeline with one stream per stage (H2D | step | D2H) chained by events."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

n = 8192
s = bx.System(open(os.path.join(ROOT, "scenes", "ant.bxc")).read())
B, A = s.n_bodies, s.act_dim
sizes = [n * B * 3, n * B * 4, n * B * 3, n * B * 3]
nq = sum(sizes)


def views(flat):
    out, o = {}, 0
    for k, sz, w in zip(("pos", "rot", "vel", "ang"), sizes, (3, 4, 3, 3)):
        out[k] = flat[o:o + sz].view(n, B, w)
        o += sz
    return out, flat[o:o + n * A].view(n, A)


qp0 = s.alloc_qp(n)
s.reset(qp0, 0, 0.1, 0.1)
act0 = torch.from_numpy(synth.actions(1, 1, n, A)[0]).cuda()
NB = 6
host_in, host_out, dflat = [], [], []
for r in range(NB):
    h = torch.empty(nq + n * A, dtype=torch.float32).pin_memory()
    hq, ha = views(h)
    for k in hq:
        hq[k].copy_(qp0[k].cpu())
    ha.copy_(act0.cpu())
    host_in.append(h)
    host_out.append(torch.empty(nq, dtype=torch.float32).pin_memory())
    dflat.append(torch.empty(nq + n * A, dtype=torch.float32, device="cuda"))
dv = [views(f) for f in dflat]
s.step(dv[0][0], dv[0][1], dv[0][0])  # autotune outside timing
torch.cuda.synchronize()
K = 200
res = {}


def timed(run, name):
    run(12)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    run(K)
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    res[name] = n * K / (e0.elapsed_time(e1) / 1e3)


for NS in (2, 3, 4, 6):
    streams = [torch.cuda.Stream() for _ in range(NS)]

    def rr(k, NS=NS, streams=streams):
        for i in range(k):
            j = i % NS
            with torch.cuda.stream(streams[j]):
                dflat[j].copy_(host_in[j], non_blocking=True)
                s.step(dv[j][0], dv[j][1], dv[j][0], stream=streams[j])
                host_out[j].copy_(dflat[j][:nq], non_blocking=True)
    timed(rr, f"roundrobin_ns{NS}")

# stage pipeline: H2D stream, compute stream, D2H stream; buffer i % NB
sh, sc, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
ev_in = [torch.cuda.Event() for _ in range(NB)]
ev_k = [torch.cuda.Event() for _ in range(NB)]
ev_out = [torch.cuda.Event() for _ in range(NB)]
started = [False] * NB


def stages(k):
    for i in range(k):
        j = i % NB
        if started[j]:
            sh.wait_event(ev_out[j])  # buffer j free once its previous result left
        with torch.cuda.stream(sh):
            dflat[j].copy_(host_in[j], non_blocking=True)
            ev_in[j].record(sh)
        sc.wait_event(ev_in[j])
        s.step(dv[j][0], dv[j][1], dv[j][0], stream=sc)
        ev_k[j].record(sc)
        sd.wait_event(ev_k[j])
        with torch.cuda.stream(sd):
            host_out[j].copy_(dflat[j][:nq], non_blocking=True)
            ev_out[j].record(sd)
        started[j] = True


timed(stages, "stages_nb6")
# host-side cost of issuing one step (no GPU wait)
import time  # noqa: E402
torch.cuda.synchronize()
t0 = time.perf_counter()
stages(50)
res["host_issue_us_per_step"] = (time.perf_counter() - t0) / 50 * 1e6
torch.cuda.synchronize()
print(json.dumps(res))
