mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep.py --scenes ant,humanoid,halfcheetah,grasp,fetch --envs 2048,4096,8192,65536 > gpurun_out/sweep_def.log 2>&1
timeout 300 python tools/phases.py --scenes ant --envs 8192 > gpurun_out/phases.log 2>&1
