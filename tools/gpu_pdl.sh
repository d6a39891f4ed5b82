# full GPU suite, the checked build on the parity / fuzz suites, then a knob
# A/B (tools/knob_ab.py "$@")
export PYTHONDONTWRITEBYTECODE=1
timeout -k 10 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/iter_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/iter_gpu.log
tail -n 2 gpurun_out/iter_gpu.log
PXR_LIB_PATH=$PWD/paper_2502_00021_b200/libpxr_checked.so timeout -k 10 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/iter_checked.log 2>&1; echo "rc=$?" >> gpurun_out/iter_checked.log
tail -n 2 gpurun_out/iter_checked.log
timeout -k 10 400 python tools/knob_ab.py "$@" > gpurun_out/knob.log 2>&1
cat gpurun_out/knob.log
