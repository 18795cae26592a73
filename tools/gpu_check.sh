#!/bin/bash
# One GPU round trip: parity tests, kernel sweep, launch list + full ncu capture of the step kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/sweep.py --scenes ant --envs 8192,32768,262144 --warps ${WARPS:-0} > gpurun_out/sweep.log 2>&1
timeout 300 python tools/sweep.py --scenes humanoid,halfcheetah,grasp,fetch --envs 4096,65536 >> gpurun_out/sweep.log 2>&1
if [ "${PROFILE:-1}" = "1" ]; then
  python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:brax_step -s 3 -c 1 -o gpurun_out/prof_${TAG:-x}_ant python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?" >> gpurun_out/ncu_full.log
fi
