# phase-stagger sweep (BRAX_STAGGER cycles), ant 8192 / 65536 at the tuned plan (2,2), 96 regs, fixed gather
mkdir -p gpurun_out
for st in 0 500 1000 1500 2000 3000 4000; do
  BRAX_STAGGER=$st BRAX_FIXED_GATHER=1 BRAX_MAXREG=96 timeout 300 python tools/sweep.py --scenes ant --envs 8192 --groups 2:2 --steps 400 | sed "s/^/stagger $st /"
done > gpurun_out/stagger.log 2>&1
for st in 0 1500 3000; do
  BRAX_STAGGER=$st timeout 300 python tools/sweep.py --scenes humanoid,halfcheetah --envs 4096 --steps 400 | sed "s/^/stagger $st /"
done >> gpurun_out/stagger.log 2>&1
