# exactness soak on the current build: 4000 fuzz seeds (product build) and
# 600 through the checked build, plus smoke()
export PYTHONDONTWRITEBYTECODE=1
PXR_FUZZ_SEEDS=4000 timeout -k 10 1500 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/soak.log 2>&1; echo "rc=$?" >> gpurun_out/soak.log
PXR_FUZZ_SEEDS=600 PXR_LIB_PATH=$PWD/paper_2502_00021_b200/libpxr_checked.so timeout -k 10 900 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/soak_checked.log 2>&1; echo "rc=$?" >> gpurun_out/soak_checked.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
for f in gpurun_out/soak.log gpurun_out/soak_checked.log gpurun_out/smoke.log; do tail -n 2 $f; done
