mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for P in 1:1 2:1 1:2 2:2 4:2; do BRAX_PLAN=${P/:/,} timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "single_step_parity or full_size" > gpurun_out/pytest_plan_${P/:/_}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_plan_${P/:/_}.log; done
timeout 900 python tools/sweep.py --scenes ant --envs 2048,8192,65536,262144 --groups 1:1,2:1,1:2,2:2,4:2 > gpurun_out/psweep.log 2>&1
timeout 600 python tools/sweep.py --scenes humanoid,halfcheetah,grasp,fetch --envs 2048,4096,65536 --groups 1:1,2:1,1:2,2:2 >> gpurun_out/psweep.log 2>&1
