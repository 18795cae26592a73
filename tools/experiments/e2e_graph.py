"""e2e pipeline (pinned host -> device -> brax_step -> host, every step) issued eagerly vs
captured once as a multi-stream CUDA graph; ant 8192."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2106_13281_b200 as bx  # noqa: E402
import synth  # noqa: E402

n, NB, K = 8192, 6, 120
s = bx.System(open(os.path.join(ROOT, "scenes", "ant.bxc")).read())
B, A = s.n_bodies, s.act_dim
sizes = [n * B * 3, n * B * 4, n * B * 3, n * B * 3]
nq = sum(sizes)
dev = torch.device("cuda", 0)


def views(flat):
    out, o = {}, 0
    for k, sz, w in zip(("pos", "rot", "vel", "ang"), sizes, (3, 4, 3, 3)):
        out[k] = flat[o:o + sz].view(n, B, w)
        o += sz
    return out, flat[o:o + n * A].view(n, A)


qp = s.alloc_qp(n)
s.reset(qp, 0, 0.1, 0.1)
act = torch.from_numpy(synth.actions(1, 1, n, A)[0]).cuda()
s.tune(qp, act)
host_in, host_out, dflat = [], [], []
for r in range(NB):
    h = torch.empty(nq + n * A, dtype=torch.float32).pin_memory()
    hq, ha = views(h)
    for k in hq:
        hq[k].copy_(qp[k].cpu())
    ha.copy_(act.cpu())
    host_in.append(h)
    host_out.append(torch.empty(nq, dtype=torch.float32).pin_memory())
    dflat.append(torch.empty(nq + n * A, dtype=torch.float32, device=dev))
dviews = [views(f) for f in dflat]
s_in, s_k, s_out, s0 = (torch.cuda.Stream() for _ in range(4))
if os.environ.get("ONECOPY"):
    s_out = s_in
ev_in = [torch.cuda.Event() for _ in range(NB)]
ev_k = [torch.cuda.Event() for _ in range(NB)]
ev_out = [torch.cuda.Event() for _ in range(NB)]


MODE = os.environ.get("MODE", "all")


def issue(i, used):
    j = i % NB
    if used[j]:
        s_in.wait_event(ev_out[j])
    with torch.cuda.stream(s_in):
        if MODE != "noh2d":
            dflat[j].copy_(host_in[j], non_blocking=True)
        ev_in[j].record(s_in)
    s_k.wait_event(ev_in[j])
    dq, da = dviews[j]
    if MODE == "sleep":
        with torch.cuda.stream(s_k):
            torch.cuda._sleep(50000)
    elif MODE != "copies":
        s.step(dq, da, dq, stream=s_k)
    ev_k[j].record(s_k)
    s_out.wait_event(ev_k[j])
    with torch.cuda.stream(s_out):
        if MODE != "nod2h":
            host_out[j].copy_(dflat[j][:nq], non_blocking=True)
        ev_out[j].record(s_out)
    used[j] = True


LAG = int(os.environ.get("LAG", "0"))


def issue_skewed(i, used):
    """iteration i: upload i, step i-LAG, download i-2*LAG (copy queue never waits on a kernel)."""
    if i < K:
        j = i % NB
        if used[j]:
            s_in.wait_event(ev_out[j])
        with torch.cuda.stream(s_in):
            dflat[j].copy_(host_in[j], non_blocking=True)
            ev_in[j].record(s_in)
    if 0 <= i - LAG < K:
        j = (i - LAG) % NB
        s_k.wait_event(ev_in[j])
        dq, da = dviews[j]
        s.step(dq, da, dq, stream=s_k)
        ev_k[j].record(s_k)
    if 0 <= i - 2 * LAG < K:
        j = (i - 2 * LAG) % NB
        s_out.wait_event(ev_k[j])
        with torch.cuda.stream(s_out):
            host_out[j].copy_(dflat[j][:nq], non_blocking=True)
            ev_out[j].record(s_out)
        used[j] = True


def eager():
    used = [False] * NB
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s0)
    for st in (s_in, s_k, s_out):
        st.wait_event(e0)
    for i in range(K + 2 * LAG):
        issue_skewed(i, used) if LAG else issue(i, used)
    s0.wait_stream(s_out)
    e1.record(s0)
    e1.synchronize()
    return e0.elapsed_time(e1)


for _ in range(2):
    eager()
ms_e = min(eager() for _ in range(3))
# graph: fork from s0, the three stage streams, join back
g = torch.cuda.CUDAGraph()
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s0):
    fork = torch.cuda.Event()
    fork.record(s0)
    for st in (s_in, s_k, s_out):
        st.wait_event(fork)
    used = [False] * NB
    for i in range(K + 2 * LAG):
        issue_skewed(i, used) if LAG else issue(i, used)
    for st in (s_in, s_k, s_out):
        s0.wait_stream(st)
g.replay()
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s0)
    with torch.cuda.stream(s0):
        g.replay()
    e1.record(s0)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
ms_g = min(ts)
print({"mode": MODE, "eager_us_per_step": 1e3 * ms_e / K, "graph_us_per_step": 1e3 * ms_g / K,
       "eager_env_steps_per_s": n * K / (ms_e / 1e3), "graph_env_steps_per_s": n * K / (ms_g / 1e3)})

# per-stage timeline (eager): event pairs around each stage of steps 20..K-20
if os.environ.get("TIMELINE"):
    T = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
         for k in ("h2d", "k", "d2h")}
    used = [False] * NB
    torch.cuda.synchronize()
    z = torch.cuda.Event(enable_timing=True)
    z.record(s0)
    for st in (s_in, s_k, s_out):
        st.wait_event(z)
    for i in range(K):
        j = i % NB
        if used[j]:
            s_in.wait_event(ev_out[j])
        T["h2d"][i][0].record(s_in)
        with torch.cuda.stream(s_in):
            dflat[j].copy_(host_in[j], non_blocking=True)
        T["h2d"][i][1].record(s_in)
        s_k.wait_event(T["h2d"][i][1])
        T["k"][i][0].record(s_k)
        dq, da = dviews[j]
        s.step(dq, da, dq, stream=s_k)
        T["k"][i][1].record(s_k)
        s_out.wait_event(T["k"][i][1])
        T["d2h"][i][0].record(s_out)
        with torch.cuda.stream(s_out):
            host_out[j].copy_(dflat[j][:nq], non_blocking=True)
        T["d2h"][i][1].record(s_out)
        ev_out[j].record(s_out)
        used[j] = True
    torch.cuda.synchronize()
    for i in range(40, 48):
        print(i, {k: (round(z.elapsed_time(v[i][0]) * 1e3, 1), round(v[i][0].elapsed_time(v[i][1]) * 1e3, 1))
                  for k, v in T.items()})
