# One build -> measure iteration on the GPU box: parity suites (both render
# kernels), then device time of the four BASELINE-shaped workloads.
set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/iter_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/iter_gpu.log
PXR_LIB_PATH=$PWD/paper_2502_00021_b200/libpxr_checked.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/iter_checked.log 2>&1; echo "rc=$?" >> gpurun_out/iter_checked.log
for m in "Humanoid video" "Walker2d video" "HalfCheetah none" "Ant color"; do
  set -- $m
  timeout 120 python tools/pipe_prof.py --model $1 --mode $2 > gpurun_out/iprof_$1.log 2>&1
done
tail -2 gpurun_out/iter_gpu.log gpurun_out/iter_checked.log
grep -h "legacy\|pipe:" gpurun_out/iprof_*.log
