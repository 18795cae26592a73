mkdir -p gpurun_out
export BRAX_PLAN=2,2 BRAX_MAXREG=96
for n in 32 8192; do
ncu --set full --clock-control none --import-source on -k regex:brax_step -s 3 -c 1 -o gpurun_out/prof_n$n python tools/profile_step.py --envs $n > gpurun_out/ncu_n$n.log 2>&1
done
