# one full ncu capture of the step kernel at ant 8192, plan (2,2), 96 registers -> gpurun_out/prof_cur.ncu-rep
mkdir -p gpurun_out
export BRAX_PLAN=${PLAN:-2,2} BRAX_MAXREG=${REGS:-96}
python tools/profile_step.py --envs ${N:-8192} > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:brax_step -s 3 -c 1 -o gpurun_out/prof_cur python tools/profile_step.py --envs ${N:-8192} > gpurun_out/ncu_cur.log 2>&1
echo rc=$? >> gpurun_out/ncu_cur.log
