mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
BRAX_PLAN=1,2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "single_step_parity or full_size" > gpurun_out/pytest_plan_1_2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_plan_1_2.log
: > gpurun_out/rsweep.log
for R in 64 80 96 112 128; do
  BRAX_MAXREG=$R timeout 300 python tools/sweep.py --scenes ant --envs 2048,8192,65536 --groups 1:1,2:1,1:2 >> gpurun_out/rsweep.log 2>&1
  BRAX_MAXREG=$R timeout 300 python tools/sweep.py --scenes humanoid,halfcheetah --envs 4096,65536 --groups 1:1,1:2 >> gpurun_out/rsweep.log 2>&1
done
