# policy timing (tools/policy_bench.py) of build/ab/libpxr_base.so against the
# working tree, plus the policy tests on the working tree
export PYTHONDONTWRITEBYTECODE=1
timeout -k 10 600 python -m pytest tests/test_policy.py tests/test_env_gpu.py -x -q -p no:cacheprovider > gpurun_out/pol_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pol_tests.log
tail -n 2 gpurun_out/pol_tests.log
for lib in build/ab/libpxr_base.so paper_2502_00021_b200/libpxr.so; do
  echo "$(basename $lib)"
  PXR_LIB_PATH=$PWD/$lib timeout 300 python tools/policy_bench.py --batches 1 10 100 500 1000 4096 16384 --iters 20 2>&1 | grep policy
done
