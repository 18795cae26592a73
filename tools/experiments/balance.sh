# one block per SM (plan G=1,V=2, E=64) at 148*64 = 9472 envs vs two per SM (plan 2,2, E=32), same envs
mkdir -p gpurun_out
for fx in 1 0; do for g in 1:2 2:2 4:2; do for r in 80 96; do
  BRAX_FIXED_GATHER=$fx BRAX_MAXREG=$r timeout 300 python tools/sweep.py --scenes ant --envs 9472,8192 --groups $g --steps 400 | sed "s/^/fx $fx g $g r $r /"
done; done; done > gpurun_out/balance.log 2>&1
