# per-warp clock stamps of the lean kernel (diagnostic build), ant 8192 / 16 at plan (4,2) and (2,2)
mkdir -p gpurun_out
BRAX_NVCC_FLAGS=-DBRAX_DIAG timeout 300 python paper_2106_13281_b200/build.py > /dev/null || exit 1
for plan in 4,2 2,2; do for n in 8192 64; do
  echo "plan $plan n=$n"
  BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_DIAG_BLOCK=1 BRAX_PLAN=$plan BRAX_MAXREG=96 timeout 120 python tools/experiments/diag_warps.py $n ant 2>&1 | grep "LEAN" | head -60
done; done > gpurun_out/diag_lean.log
