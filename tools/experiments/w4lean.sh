# ant 8192 plan (4,2): lean W = 5 (one item step per warp) vs W = 4 (one warp with two) at 96 / 128 registers
mkdir -p gpurun_out
for rep in 1 2; do
  BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_MAXREG=96 timeout 300 python tools/sweep.py --scenes ant --envs 8192,65536 --steps 400 --groups 4:2 | sed "s/^/W5-r96 /"
  for r in 96 128; do
    BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_MAXREG=$r timeout 300 python tools/sweep.py --scenes ant --envs 8192,65536 --steps 400 --groups 4:2 --warps 4 | sed "s/^/W4-r$r /"
  done
  BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_MAXREG=96 timeout 300 python tools/sweep.py --scenes halfcheetah,humanoid --envs 4096 --steps 400 --groups 4:2 | sed "s/^/dflt-r96 /"
  BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_MAXREG=128 timeout 300 python tools/sweep.py --scenes halfcheetah --envs 4096 --steps 400 --groups 4:2 --warps 4 | sed "s/^/W4-r128 /"
  BRAX_LEAN=1 BRAX_FIXED_GATHER=1 BRAX_MAXREG=128 timeout 300 python tools/sweep.py --scenes humanoid --envs 4096 --steps 400 --groups 4:2 --warps 8 | sed "s/^/W8-r128 /"
done > gpurun_out/w4lean.log 2>&1
