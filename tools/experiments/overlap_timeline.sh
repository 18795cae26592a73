# block timelines of consecutive overlapped launches (diagnostic build in _ab/libdiag.so):
# ant 8192, 8 in-place launches captured in a graph, each tagged through BRAX_DIAG_BLOCK;
# every block's entry / after-wait / staged / loop-end / stored / exit times (globaltimer)
mkdir -p gpurun_out
cat > /tmp/otl.py <<'PY'
import ctypes, os, sys, torch
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2106_13281_b200 as bx, synth
s = bx.System(open("scenes/ant.bxc").read())
n, K = 8192, 8
q = s.alloc_qp(n)
s.reset(q, 0, 0.1, 0.1)
acts = torch.from_numpy(synth.actions(1, K, n, s.act_dim)).cuda()
for i in range(K): s.step(q, acts[i], q)
torch.cuda.synchronize()
st = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for i in range(K):
        os.environ["BRAX_DIAG_BLOCK"] = str(1000 + i)
        s.step(q, acts[i], q)
os.environ.pop("BRAX_DIAG_BLOCK")
torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
buf = np.zeros(16 * 4096 * 8, dtype=np.int64)
assert bx.lib.brax_diag_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_longlong(buf.size)) == 0
tl = buf.reshape(16, 4096, 8)[:K, :n // 16]
t0 = tl[:, :, 0][tl[:, :, 0] > 0].min()
print("launch overlap  start(us) first/median/last   data-ready(us) median   end(us) first/median/last   wait(us) median/max")
for k in range(K):
    r = tl[k]
    st0, ready, end = (r[:, 0] - t0) / 1e3, (r[:, 1] - t0) / 1e3, (r[:, 7] - t0) / 1e3
    w = (r[:, 1] - r[:, 0]) / 1e3
    print(f"{k:6d} {int(r[0, 6]):7d}  {st0.min():7.1f} {np.median(st0):7.1f} {st0.max():7.1f}   {np.median(ready):7.1f}"
          f"   {end.min():7.1f} {np.median(end):7.1f} {end.max():7.1f}   {np.median(w):6.1f} {w.max():6.1f}")
ph = np.concatenate([tl[k] for k in range(1, K)])
print("median per block (us): wait %.2f  stage %.2f  loop %.2f  store %.2f  release+exit %.2f" % tuple(
    np.median((ph[:, b] - ph[:, a]) / 1e3) for a, b in ((0, 1), (1, 2), (2, 3), (3, 4), (4, 7))))
tot = (tl[K - 1, :, 7].max() - t0) / 1e3
print(f"{K} launches in {tot:.1f} us: {tot / K:.2f} us per launch")
PY
BRAX_LIB_PATH=$PWD/_ab/${DIAGLIB:-libdiag.so} BRAX_PLAN=4,2 BRAX_MAXREG=96 BRAX_FIXED_GATHER=1 BRAX_LEAN=1 timeout 120 python /tmp/otl.py > gpurun_out/overlap_timeline.txt 2>&1
