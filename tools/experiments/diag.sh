# per-warp clock stamps (diagnostic build), lone block (32 envs): ant vs ant without capsule contacts
mkdir -p gpurun_out
BRAX_NVCC_FLAGS=-DBRAX_DIAG python paper_2106_13281_b200/build.py > /dev/null || exit 1
for sc in ant tools/experiments/scenes/ant_nocap.bxc; do
echo "scene=$sc"
BRAX_DIAG_BLOCK=1 BRAX_PLAN=2,2 BRAX_MAXREG=96 python tools/experiments/diag_warps.py 32 $sc 2>&1 | grep "DIAG sm" | head -45
done > gpurun_out/diag.log
