# Pipelined render kernel: parity suites forced through it (several envs per
# CTA at small batches), then the default dispatch, then a short bench.
set -x
export PYTHONDONTWRITEBYTECODE=1
PXR_DEBUG_RENDER=pipe PXR_DEBUG_GRID=5 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/pipe_forced.log 2>&1; echo "rc=$?" >> gpurun_out/pipe_forced.log
PXR_LIB_PATH=$PWD/paper_2502_00021_b200/libpxr_checked.so PXR_DEBUG_RENDER=pipe PXR_DEBUG_GRID=5 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "golden or replay or round" > gpurun_out/pipe_checked.log 2>&1; echo "rc=$?" >> gpurun_out/pipe_checked.log
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/pipe_bench.log 2>&1; echo "rc=$?" >> gpurun_out/pipe_bench.log
PXR_DEBUG_RENDER=legacy timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/legacy_bench.log 2>&1; echo "rc=$?" >> gpurun_out/legacy_bench.log
tail -3 gpurun_out/pipe_forced.log gpurun_out/pipe_checked.log
grep -o '"ms_per_step": [0-9.]*' gpurun_out/pipe_bench.log gpurun_out/legacy_bench.log
