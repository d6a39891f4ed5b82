export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/small_batch.py > gpurun_out/small_batch.log 2>&1; echo "rc=$?" >> gpurun_out/small_batch.log
timeout 300 python -m pytest tests/test_physics_api.py -q -p no:cacheprovider > gpurun_out/phys3.log 2>&1; echo "rc=$?" >> gpurun_out/phys3.log
cmd="python tools/prof_step.py --model HalfCheetah --mode none --envs 1 --steps 4 --timed 4"
$cmd > gpurun_out/b1_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:render_step -s 5 -c 1 -o gpurun_out/r2_halfcheetah_none_b1 $cmd > gpurun_out/b1_ncu.log 2>&1
cat gpurun_out/small_batch.log; tail -2 gpurun_out/phys3.log
