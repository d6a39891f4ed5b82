# parity subset on the working-tree build and on build/ab/libpxr_$1.so, then
# an interleaved A/B/C of build/ab/libpxr_base.so, the working tree and
# build/ab/libpxr_$1.so over the four BASELINE workloads
export PYTHONDONTWRITEBYTECODE=1
c=${1:-variant}
timeout -k 10 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
PXR_LIB_PATH=$PWD/build/ab/libpxr_$c.so timeout -k 10 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/q_tests_c.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests_c.log
for f in gpurun_out/q_tests.log gpurun_out/q_tests_c.log; do tail -n 2 $f; done
for i in 1 2; do
  for lib in build/ab/libpxr_base.so paper_2502_00021_b200/libpxr.so build/ab/libpxr_$c.so; do
    for m in "Humanoid video" "HalfCheetah none" "Walker2d video" "Ant color"; do
      set -- $m
      echo -n "$(basename "$lib") "
      PXR_LIB_PATH=$PWD/$lib timeout 120 python tools/prof_step.py --timed 50 --model "$1" --mode "$2" | tail -1
    done
  done
done
for lib in build/ab/libpxr_base.so paper_2502_00021_b200/libpxr.so build/ab/libpxr_$c.so; do
  echo "$(basename "$lib")"
  PXR_LIB_PATH=$PWD/$lib timeout 120 python tools/phase_prof.py --cases HalfCheetah:none:1 Humanoid:video:1 Walker2d:video:100 2>&1 | grep "us/launch"
done
