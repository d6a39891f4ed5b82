# One build -> measure iteration on the GPU box: parity suites, the checked
# build on the parity / fuzz suites, then per-phase cycles and graph-replay
# device time of the BASELINE-shaped workloads.
export PYTHONDONTWRITEBYTECODE=1
timeout -k 10 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/iter_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/iter_gpu.log
PXR_LIB_PATH=$PWD/paper_2502_00021_b200/libpxr_checked.so timeout -k 10 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/iter_checked.log 2>&1; echo "rc=$?" >> gpurun_out/iter_checked.log
timeout -k 10 300 python tools/phase_prof.py --cases ${PROF_CASES:-HalfCheetah:none:1 Humanoid:video:1 HalfCheetah:none:10 Walker2d:video:100 Humanoid:video:4096 Walker2d:video:4096 HalfCheetah:none:4096 Ant:color:1024} > gpurun_out/iter_prof.log 2>&1
tail -2 gpurun_out/iter_gpu.log; tail -2 gpurun_out/iter_checked.log; grep "us/launch" gpurun_out/iter_prof.log
