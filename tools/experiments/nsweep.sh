# M6 N-sweep: ant at 1k..256k envs, tuned; the other scenes at 4k / 65k
mkdir -p gpurun_out
timeout 600 python tools/sweep.py --scenes ant --envs 1024,2048,4096,8192,16384,65536,262144 --steps 200 > gpurun_out/nsweep.jsonl 2>&1
timeout 600 python tools/sweep.py --scenes humanoid,halfcheetah,grasp,fetch --envs 4096,65536 --steps 200 >> gpurun_out/nsweep.jsonl 2>&1
