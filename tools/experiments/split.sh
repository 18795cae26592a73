# lean-kernel body splits: ant / humanoid / halfcheetah / fetch / grasp, split count 0, 1, 2, 3 (min cost 3)
mkdir -p gpurun_out
for sp in 0 1 2 3; do
  BRAX_SPLIT_MAX=$sp BRAX_SPLIT_MIN_COST=3 timeout 300 python tools/sweep.py --scenes ant --envs 8192 --steps 400 | sed "s/^/split $sp /"
  BRAX_SPLIT_MAX=$sp BRAX_SPLIT_MIN_COST=3 timeout 300 python tools/sweep.py --scenes humanoid,halfcheetah --envs 4096 --steps 400 | sed "s/^/split $sp /"
  BRAX_SPLIT_MAX=$sp BRAX_SPLIT_MIN_COST=3 timeout 300 python tools/sweep.py --scenes grasp,fetch --envs 2048 --steps 400 | sed "s/^/split $sp /"
done > gpurun_out/split.log 2>&1
