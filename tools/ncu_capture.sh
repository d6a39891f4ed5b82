#!/usr/bin/env bash
# One `ncu --set full` capture of a steady-state render launch of a workload
# (tools/prof_step.py), after the same command has exited 0 without ncu.
# usage: bash tools/ncu_capture.sh <tag> <model> <mode> <envs>
set -u
tag=$1; model=$2; mode=$3; envs=$4
cmd="python tools/prof_step.py --model $model --mode $mode --envs $envs --steps 4 --timed 4"
$cmd > gpurun_out/${tag}_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:render_step -s 5 -c 1 \
    -o gpurun_out/${tag} $cmd > gpurun_out/${tag}_ncu.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/${tag}_plain.log
