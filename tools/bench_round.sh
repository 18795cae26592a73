#!/bin/bash
# Driver-equivalent bench runs + the ncu launch list of the same command (one GPU).
#   TAG=r2a bash tools/bench_round.sh
# Writes gpurun_out/{bench20,bench,bench_ref,launches,smoke}_${TAG}.*
TAG=${TAG:-r2}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_${TAG}.csv 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
CMD20="python bench.py --gpus 1 --steps 20 --warmup 5"
timeout 900 $CMD20 > gpurun_out/bench20_${TAG}.json 2> gpurun_out/bench20_${TAG}.err; echo "rc=$?" >> gpurun_out/bench20_${TAG}.err
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "rc=$?" >> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
# the driver's multi-GPU launcher at N = 1 (torchrun, NCCL communicator of one rank)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_tr_${TAG}.json 2> gpurun_out/bench_tr_${TAG}.err
# launch list of the driver's command (no scenes / env / vjp: the same timed region, fewer other kernels),
# with the launch configuration the bench tuned pinned (ncu's serialised replay distorts the tuner's timings)
kc() { python -c "import json; c=json.loads([l for l in open('gpurun_out/bench20_${TAG}.json') if l.startswith('{')][0])['config']['kernel_config']; print($1)" 2>/dev/null; }
export BRAX_PLAN=$(kc "f\"{c['G']},{c['V']}\"") BRAX_MAXREG=$(kc "c['regs']") BRAX_FIXED_GATHER=$(kc "c['fixed_gather']") BRAX_LEAN=$(kc "c['lean']")
echo "pinned plan $BRAX_PLAN regs $BRAX_MAXREG fixed $BRAX_FIXED_GATHER lean $BRAX_LEAN" > gpurun_out/pinned_${TAG}.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-scenes --no-env --no-rollout --no-vjp --e2e-steps 6 \
  > gpurun_out/ncu_launch_${TAG}.log 2>&1
# one full capture of the step kernel the bench timed (same pinned configuration)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:brax_step -s 3 -c 1 -o gpurun_out/prof_${TAG} \
  python tools/profile_step.py > gpurun_out/ncu_full_${TAG}.log 2>&1
unset BRAX_PLAN BRAX_MAXREG BRAX_FIXED_GATHER BRAX_LEAN
echo done
