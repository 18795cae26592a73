# NEXT-2 cost: brax_step vs brax_rollout (T steps per launch), ant 8192
mkdir -p gpurun_out
for r in 0 10 100; do timeout 300 python tools/sweep.py --scenes ant --envs 8192 --rollout $r --steps 200 | cut -c1-260; done > gpurun_out/rollout.log 2>&1
