# parity subset on the working-tree build, then an interleaved A/B against
# build/ab/libpxr_base.so (tools/build_base.sh) over the four BASELINE workloads
export PYTHONDONTWRITEBYTECODE=1
timeout -k 10 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
tail -2 gpurun_out/q_tests.log
timeout -k 10 400 bash tools/ab4.sh build/ab/libpxr_base.so paper_2502_00021_b200/libpxr.so 2 > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
