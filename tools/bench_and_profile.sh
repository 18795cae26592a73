#!/bin/bash
# bench.py (N=1) + reference arm + ncu launch list of the same bench command + one full
# ncu capture of the step kernel.  Writes gpurun_out/{bench,bench_ref,launches,ncu}.*
# The launch list and the capture pin the launch configuration the bench's autotuner
# chose (BRAX_PLAN / BRAX_MAXREG / BRAX_FIXED_GATHER): under ncu's serialised replay the
# autotuner's own timings are distorted and could pick another variant.
TAG=${TAG:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_${TAG}.csv 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 200 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
kc() { python -c "import json; c=json.load(open('gpurun_out/bench_${TAG}.json'))['config']['kernel_config']; print($1)" 2>/dev/null; }
PLAN=$(kc "f\"{c['G']},{c['V']}\"") ; PLAN=${PLAN:-1,1}
REGS=$(kc "c['regs']") ; REGS=${REGS:-96}
FIXED=$(kc "c.get('fixed_gather', 0)") ; FIXED=${FIXED:-0}
export BRAX_PLAN=$PLAN BRAX_MAXREG=$REGS BRAX_FIXED_GATHER=$FIXED
CMD="python bench.py --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 2 --no-env --no-vjp"
$CMD > gpurun_out/bench_small_${TAG}.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
python tools/profile_step.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:brax_step -s 3 -c 1 -o gpurun_out/prof_${TAG}_ant python tools/profile_step.py > gpurun_out/ncu_full_${TAG}.log 2>&1
unset BRAX_PLAN BRAX_MAXREG BRAX_FIXED_GATHER
echo "done (plan $PLAN, regs $REGS, fixed gather $FIXED)"
