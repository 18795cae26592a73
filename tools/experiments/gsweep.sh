mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep.py --scenes ant --envs 2048,8192,16384,65536,262144 --groups 1,2,4 > gpurun_out/gsweep.log 2>&1
timeout 600 python tools/sweep.py --scenes humanoid,halfcheetah,grasp,fetch --envs 2048,4096 --groups 1,2,4 >> gpurun_out/gsweep.log 2>&1
