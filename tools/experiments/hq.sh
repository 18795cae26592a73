mkdir -p gpurun_out
for fx in 0 1; do for g in 1:2 2:2; do BRAX_FIXED_GATHER=$fx BRAX_MAXREG=128 timeout 120 python tools/sweep.py --scenes humanoid --envs 8192 --groups $g --steps 200 | sed "s/^/fx=$fx /"; done; done > gpurun_out/hq.log 2>&1
BRAX_MAXREG=64 timeout 120 python tools/sweep.py --scenes humanoid --envs 8192 --groups 1:1 --steps 200 | sed "s/^/fx=0 /" >> gpurun_out/hq.log 2>&1
