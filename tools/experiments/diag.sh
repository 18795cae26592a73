mkdir -p gpurun_out
for n in 8192 32; do
BRAX_DIAG_BLOCK=1 BRAX_PLAN=2,2 BRAX_MAXREG=96 python tools/experiments/diag_warps.py $n ant 2>&1 | grep -v "^$" | sort | uniq | head -60
done > gpurun_out/diag.log
