# one item / body per warp with G = 1 (W = 17 for ant): lean kernel at 9472 = 148 x 64 and 8192 envs
mkdir -p gpurun_out
for w in 17 18; do for r in 96 128; do
  BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_MAXREG=$r timeout 300 python tools/sweep.py --scenes ant --envs 9472,8192 --groups 1:2 --warps $w --steps 400 | sed "s/^/W $w r $r /"
done; done > gpurun_out/g1.log 2>&1
# | sed "s/^/tuned /" >> gpurun_out/g1.log 2>&1
