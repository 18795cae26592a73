mkdir -p gpurun_out; : > gpurun_out/wsweep2.log
timeout 600 python tools/sweep.py --scenes ant --envs 2048,8192,65536 --groups 1:1,2:1 --warps 8,9,10,12,13,16 >> gpurun_out/wsweep2.log 2>&1
timeout 300 python tools/sweep.py --scenes humanoid --envs 2048,4096 --groups 1:1,2:1 --warps 8,11,12,14,16 >> gpurun_out/wsweep2.log 2>&1
