# quick A/B: parity subset + graph-replay timing of the BASELINE-shaped workloads
export PYTHONDONTWRITEBYTECODE=1
timeout -k 10 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout -k 10 180 python tools/phase_prof.py --cases ${PROF_CASES:-Humanoid:video:4096 Walker2d:video:4096 HalfCheetah:none:4096 Ant:color:1024 HalfCheetah:none:1} > gpurun_out/q_prof.log 2>&1
tail -2 gpurun_out/q_tests.log; grep "us/launch" gpurun_out/q_prof.log
