# fixed vs per-substep cost: ant 8192 with the substep count overridden (tuned plan each)
mkdir -p gpurun_out
for S in 1 2 5 10 20; do
  timeout 300 python tools/sweep.py --scenes ant --envs 8192 --substeps $S --steps 400 | sed "s/^/S $S /"
done > gpurun_out/substeps.log 2>&1
