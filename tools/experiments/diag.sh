# per-warp clock stamps (diagnostic build), ant, specialised variant, plan (2,2)
mkdir -p gpurun_out
BRAX_NVCC_FLAGS=-DBRAX_DIAG python paper_2106_13281_b200/build.py > /dev/null || exit 1
for n in 32 8192; do
echo "n=$n"
BRAX_FIXED_GATHER=1 BRAX_DIAG_BLOCK=1 BRAX_PLAN=2,2 BRAX_MAXREG=96 python tools/experiments/diag_warps.py $n ant 2>&1 | grep "DIAG" | head -${LINES_PER:-120}
done > gpurun_out/diag.log
