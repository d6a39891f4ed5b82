cmd="python tools/prof_step.py --model HalfCheetah --mode none --envs 1 --steps 4 --timed 4"
$cmd > gpurun_out/b1_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:render_step -s 5 -c 3 -o gpurun_out/r2_b1_dense $cmd > gpurun_out/b1_ncu.log 2>&1
echo rc=$?
