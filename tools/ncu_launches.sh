# the bench command's launch list under ncu (serialised, cold caches: compare
# shares, not absolutes), after the same command exited 0 without ncu
cmd="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$cmd > gpurun_out/launches_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r2_launches_humanoid_video_4096.csv $cmd > gpurun_out/launches_ncu.log 2>&1
echo rc=$?
