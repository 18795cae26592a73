# warps per block x register budget for the specialised (fixed-gather) variant, ant 8192, plan (2,2)
mkdir -p gpurun_out
for W in 9 10 11 12; do for R in 80 96; do
  BRAX_FIXED_GATHER=1 BRAX_MAXREG=$R timeout 120 python tools/sweep.py --scenes ant --envs 8192 --warps $W --groups 2:2 --steps 200 2>&1 | sed "s/^/W=$W R=$R /"
done; done > gpurun_out/wsweep2.log
