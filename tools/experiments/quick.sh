# quick kernel timing: ant 8192 / 65536 autotuned, then forced (G,V) = (2,2) at 96 registers; + gpu tests
mkdir -p gpurun_out
timeout 300 python tools/sweep.py --scenes ant --envs 8192,65536 --steps 200 > gpurun_out/quick.log 2>&1
BRAX_MAXREG=96 timeout 300 python tools/sweep.py --scenes ant,humanoid,grasp --envs 8192 --groups 2:2 --steps 200 >> gpurun_out/quick.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/quick_pt.log 2>&1; tail -2 gpurun_out/quick_pt.log | sed 's/^/PT /' >> gpurun_out/quick.log
