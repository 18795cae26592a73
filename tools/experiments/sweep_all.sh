# autotuned throughput of every scene at 2k / 4k / 8k / 64k envs (kernel characterisation)
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --scenes ant,humanoid,halfcheetah,grasp,fetch,pendulum,chain2,ball --envs 2048,4096,8192,65536 --steps 200 > gpurun_out/sweep_autotune.jsonl 2> gpurun_out/sweep_autotune.err
