mkdir -p gpurun_out
for R in 80 96 128; do
BRAX_MAXREG=$R timeout 120 python tools/sweep.py --scenes ant --envs 32,1024,4096,8192 --groups 2:2,2:1 --steps 100 2>&1 | sed "s/^/R=$R /"
done > gpurun_out/regs_lone.log
