# launch overlap (granule protocol) vs the grid-wide PDL wait: ant 8192 and the other scenes
mkdir -p gpurun_out
for rep in 1 2; do
  for ov in 1 0; do
    if [ $ov = 0 ]; then export BRAX_NO_OVERLAP=1; else unset BRAX_NO_OVERLAP; fi
    for sn in ant:8192 humanoid:4096 halfcheetah:4096 grasp:2048 fetch:2048 ant:65536; do
      sc=${sn%%:*}; n=${sn##*:}
      timeout 300 python tools/sweep.py --scenes $sc --envs $n --steps 400 | sed "s/^/overlap$ov rep$rep /"
    done
  done
done > gpurun_out/overlap.log 2>&1
