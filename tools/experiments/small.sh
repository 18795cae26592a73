# small batches (grasp / fetch 2048): every plan, lean on/off, 96/128 registers
mkdir -p gpurun_out
for sc in grasp fetch; do
  for g in 2:1 4:1 2:2 4:2 1:1; do
    for lean in 0 1; do
      for r in 96 128; do
        BRAX_LEAN=$lean BRAX_FIXED_GATHER=$lean BRAX_MAXREG=$r timeout 120 python tools/sweep.py --scenes $sc --envs 2048 --steps 200 --groups $g 2>/dev/null | sed "s/^/$sc g$g lean$lean r$r /"
      done
    done
  done
done > gpurun_out/small.log 2>&1
