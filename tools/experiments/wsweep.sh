mkdir -p gpurun_out
for W in 8 9 10 12; do for R in 80 96 128; do
  BRAX_MAXREG=$R timeout 120 python tools/sweep.py --scenes ant --envs 8192,65536 --warps $W --groups 2:2,1:2 --steps 200 2>&1 | sed "s/^/W=$W R=$R /"
done; done > gpurun_out/wsweep.log
