set -x
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_env_gpu.py tests/test_physics_api.py tests/test_recorder.py tests/test_gpu_fullsize.py tests/test_gpu_physics_props.py -q -p no:cacheprovider > gpurun_out/phys_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/phys_tests2.log
timeout 600 python tools/pose_validation.py > gpurun_out/pose_validation.md 2> gpurun_out/pose_validation.err
tail -5 gpurun_out/phys_tests2.log; cat gpurun_out/pose_validation.md; tail -3 gpurun_out/pose_validation.err
