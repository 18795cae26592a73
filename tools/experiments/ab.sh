# A/B timing of two library builds (_ab/libA.so, _ab/libB.so) in one box session, alternating.
#   SCENES="ant:8192" ARGS="--groups 2:2" bash tools/experiments/ab.sh
mkdir -p gpurun_out
SCENES=${SCENES:-"ant:8192 humanoid:4096 halfcheetah:4096 grasp:2048 fetch:2048"}
for rep in 1 2 3; do
  for lib in ${LIBS:-A B}; do
    for sn in $SCENES; do
      sc=${sn%%:*}; n=${sn##*:}
      BRAX_LIB_PATH=$PWD/_ab/lib$lib.so timeout 300 python tools/sweep.py --scenes $sc --envs $n --steps 400 $ARGS | sed "s/^/$lib rep$rep /"
    done
  done
done > gpurun_out/ab${TAG}.log 2>&1
