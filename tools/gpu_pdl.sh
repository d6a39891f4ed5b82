export PYTHONDONTWRITEBYTECODE=1
timeout -k 10 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/iter_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/iter_gpu.log
tail -n 2 gpurun_out/iter_gpu.log
timeout -k 10 400 python tools/pdl_ab.py > gpurun_out/pdl.log 2>&1
cat gpurun_out/pdl.log
