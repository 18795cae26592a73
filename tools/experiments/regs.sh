# ant 8192: tuned plan, and plan (2,2) fixed at 80/96/112/128 registers
mkdir -p gpurun_out
( timeout 300 python tools/sweep.py --scenes ant --envs 8192 --steps 400 | sed 's/^/tuned /'
for r in 96 112 128; do BRAX_FIXED_GATHER=1 BRAX_MAXREG=$r timeout 300 python tools/sweep.py --scenes ant --envs 8192 --groups 2:2 --steps 400 | sed "s/^/r $r /"; done
timeout 300 python tools/sweep.py --scenes humanoid,halfcheetah --envs 4096 --steps 400 | sed 's/^/tuned /'
timeout 300 python tools/sweep.py --scenes grasp,fetch --envs 2048 --steps 400 | sed 's/^/tuned /' ) > gpurun_out/regs.log 2>&1
