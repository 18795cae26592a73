# block timelines of the lean kernel (diagnostic build): ant 8192, 4 consecutive launches
mkdir -p gpurun_out
BRAX_NVCC_FLAGS=-DBRAX_DIAG timeout 300 python paper_2106_13281_b200/build.py > /dev/null || exit 1
cat > /tmp/tl.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2106_13281_b200 as bx, synth
s = bx.System(open("scenes/ant.bxc").read())
n = 8192
qs = [s.alloc_qp(n) for _ in range(4)]
for q in qs: s.reset(q, 0, 0.1, 0.1)
acts = torch.from_numpy(synth.actions(1, 4, n, s.act_dim)).cuda()
os.environ.pop("BRAX_DIAG_BLOCK", None)
for i in range(8): s.step(qs[i % 4], acts[i % 4], qs[i % 4])
torch.cuda.synchronize()
os.environ["BRAX_DIAG_BLOCK"] = "1"
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(4): s.step(qs[i], acts[i], qs[i])
torch.cuda.synchronize()
print("replay", flush=True)
g.replay(); torch.cuda.synchronize()
PY
BRAX_PLAN=4,2 BRAX_MAXREG=96 BRAX_FIXED_GATHER=1 BRAX_LEAN=1 timeout 120 python /tmp/tl.py > gpurun_out/timeline.log 2>&1
