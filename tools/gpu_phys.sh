set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python tools/physics_exact.py > gpurun_out/phys_exact.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_env_gpu.py tests/test_physics_api.py tests/test_recorder.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -s > gpurun_out/phys_tests.log 2>&1; echo "rc=$?" >> gpurun_out/phys_tests.log
cat gpurun_out/phys_exact.log | tail -50; tail -5 gpurun_out/phys_tests.log
