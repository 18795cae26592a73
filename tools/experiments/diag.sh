# per-warp clock stamps (diagnostic build in a scratch copy of the library)
mkdir -p gpurun_out
BRAX_NVCC_FLAGS=-DBRAX_DIAG python paper_2106_13281_b200/build.py > /dev/null || exit 1
for n in 32 8192; do
echo "n=$n"
BRAX_DIAG_BLOCK=1 BRAX_PLAN=2,2 BRAX_MAXREG=96 python tools/experiments/diag_warps.py $n ant 2>&1 | grep DIAG | head -${LINES_PER:-30}
done > gpurun_out/diag.log
