# A/B against HEAD plus a 1000-seed fuzz soak of the working-tree build
export PYTHONDONTWRITEBYTECODE=1
PXR_FUZZ_SEEDS=1000 timeout -k 10 600 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
tail -n 2 gpurun_out/q_tests.log
timeout -k 10 400 bash tools/ab4.sh build/ab/libpxr_base.so paper_2502_00021_b200/libpxr.so 2 > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
