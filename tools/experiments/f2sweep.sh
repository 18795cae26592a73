# GPU tests, bitwise plan check, autotuned sweep, bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/plan_bits.py > gpurun_out/plan_bits.log 2>&1
timeout 900 python tools/sweep.py --scenes ant,humanoid,halfcheetah,grasp,fetch --envs 2048,8192,65536 > gpurun_out/tunesweep.log 2>&1
timeout 900 python tools/sweep.py --scenes ant --envs 8192 --groups 1:1,2:1,1:2,2:2,4:2 >> gpurun_out/tunesweep.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_tune.json 2> gpurun_out/bench_tune.err
