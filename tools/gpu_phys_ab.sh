# physics step timing (tools/step_split.py) of build/ab/libpxr_base.so against the
# working tree, plus the physics / env parity tests on the working tree
export PYTHONDONTWRITEBYTECODE=1
timeout -k 10 600 python -m pytest tests/test_physics_api.py tests/test_env_gpu.py tests/test_recorder.py -x -q -p no:cacheprovider > gpurun_out/phys_tests.log 2>&1; echo "rc=$?" >> gpurun_out/phys_tests.log
tail -n 2 gpurun_out/phys_tests.log
for lib in build/ab/libpxr_base.so paper_2502_00021_b200/libpxr.so; do
  for m in humanoid_lite cheetah_lite; do
    for b in 1 100 1000 2048 4096; do
      echo -n "$(basename $lib) "
      PXR_LIB_PATH=$PWD/$lib timeout 120 python tools/step_split.py --model $m --envs $b 2>&1 | tail -1
    done
  done
done
