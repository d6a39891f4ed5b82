set -x
export PYTHONDONTWRITEBYTECODE=1
for m in "Humanoid video" "Walker2d video" "HalfCheetah none" "Ant color"; do
  set -- $m
  timeout 120 python tools/pipe_prof.py --model $1 --mode $2 > gpurun_out/prof_$1.log 2>&1
  for g in 8 16; do
    PXR_LIB_PATH=$PWD/build/var/libpxr_gw$g.so timeout 120 python tools/pipe_prof.py --model $1 --mode $2 > gpurun_out/prof_$1_gw$g.log 2>&1
  done
done
PXR_DEBUG_RENDER=pipe PXR_DEBUG_GRID=5 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/pipe_forced.log 2>&1; echo "rc=$?" >> gpurun_out/pipe_forced.log
tail -2 gpurun_out/pipe_forced.log
