# one full ncu capture of the lean step kernel at ant 8192 (plan from env, default 4,2 / 96 regs)
mkdir -p gpurun_out
export BRAX_PLAN=${PLAN:-4,2} BRAX_MAXREG=${REGS:-96} BRAX_FIXED_GATHER=1 BRAX_LEAN=1
python tools/profile_step.py --envs ${N:-8192} > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:brax_step -s 3 -c 1 -o gpurun_out/prof_${TAG:-lean} python tools/profile_step.py --envs ${N:-8192} > gpurun_out/ncu_${TAG:-lean}.log 2>&1
echo rc=$? >> gpurun_out/ncu_${TAG:-lean}.log
