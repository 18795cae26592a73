# per-launch time vs graph length K (pipeline fill / drain of overlapped launches)
mkdir -p gpurun_out
for K in 5 10 20 40 100 400 2000; do
  timeout 300 python bench.py --steps $K --warmup 5 --no-cpu-baseline --no-scenes --no-env --no-rollout --no-vjp --e2e-steps 4 | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print($K, round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3))"
done > gpurun_out/ksweep.txt 2>&1
