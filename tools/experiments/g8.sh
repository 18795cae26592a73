# G = 8 plans (four lanes per group) at the small-batch configurations, lean and generic
mkdir -p gpurun_out
for sn in grasp:2048 fetch:2048 humanoid:4096 halfcheetah:4096 ant:4096 ant:8192; do
  sc=${sn%%:*}; n=${sn##*:}
  timeout 300 python tools/sweep.py --scenes $sc --envs $n --steps 300 | sed "s/^/tuned /"
  for g in 8:1 8:2; do
    for lean in 0 1; do
      BRAX_LEAN=$lean BRAX_FIXED_GATHER=$lean BRAX_MAXREG=128 timeout 300 python tools/sweep.py --scenes $sc --envs $n --steps 300 --groups $g 2>/dev/null | sed "s/^/g$g lean$lean /"
    done
  done
done > gpurun_out/g8.log 2>&1
