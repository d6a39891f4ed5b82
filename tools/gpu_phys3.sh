export PYTHONDONTWRITEBYTECODE=1
timeout 600 python tools/physics_exact.py > gpurun_out/phys_exact2.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/iter_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/iter_gpu.log
tail -3 gpurun_out/iter_gpu.log; grep "reset qvel\|chain" gpurun_out/phys_exact2.log
