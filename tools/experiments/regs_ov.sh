# register budget of the lean (4,2) kernel under launch overlap, ant 8192 / 16384 / 65536
mkdir -p gpurun_out
for r in 80 96 128; do
  BRAX_PLAN=4,2 BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_MAXREG=$r timeout 300 python tools/sweep.py --scenes ant --envs 8192,16384,65536 --steps 400 --groups 4:2 | sed "s/^/r$r /"
done > gpurun_out/regs_ov.log 2>&1
