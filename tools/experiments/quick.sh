# quick kernel timing: ant 8192 / 65536 autotuned; forced (2,2)/96 for ant, humanoid, grasp; autotuned 5 scenes at 8192
mkdir -p gpurun_out
timeout 300 python tools/sweep.py --scenes ant --envs 8192,65536 --steps 200 > gpurun_out/quick.log 2>&1
BRAX_FIXED_GATHER=1 BRAX_MAXREG=96 timeout 300 python tools/sweep.py --scenes ant,humanoid,grasp --envs 8192 --groups 2:2 --steps 200 >> gpurun_out/quick.log 2>&1
timeout 300 python tools/sweep.py --scenes humanoid,halfcheetah,grasp,fetch --envs 4096,8192 --steps 200 | sed 's/^/auto /' >> gpurun_out/quick.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/quick_pt.log 2>&1; tail -2 gpurun_out/quick_pt.log | sed 's/^/PT /' >> gpurun_out/quick.log
