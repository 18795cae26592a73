# ant 8192, plan (4,2): W = 5 warps at 96 registers vs W = 4 (one warp takes two item steps) at 128
mkdir -p gpurun_out
for rep in 1 2; do
  BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_MAXREG=96 timeout 300 python tools/sweep.py --scenes ant --envs 8192 --steps 400 --groups 4:2 | sed "s/^/lean-W5-r96 /"
  BRAX_LEAN=0 BRAX_FIXED_GATHER=1 BRAX_MAXREG=96 timeout 300 python tools/sweep.py --scenes ant --envs 8192 --steps 400 --groups 4:2 | sed "s/^/gen-W5-r96 /"
  BRAX_LEAN=0 BRAX_FIXED_GATHER=1 BRAX_MAXREG=128 timeout 300 python tools/sweep.py --scenes ant --envs 8192 --steps 400 --groups 4:2 --warps 4 | sed "s/^/gen-W4-r128 /"
  BRAX_LEAN=0 BRAX_FIXED_GATHER=1 BRAX_MAXREG=96 timeout 300 python tools/sweep.py --scenes ant --envs 8192 --steps 400 --groups 4:2 --warps 4 | sed "s/^/gen-W4-r96 /"
  BRAX_LEAN=0 BRAX_FIXED_GATHER=1 BRAX_MAXREG=128 timeout 300 python tools/sweep.py --scenes ant --envs 8192 --steps 400 --groups 4:2 | sed "s/^/gen-W5-r128 /"
done > gpurun_out/w4.log 2>&1
