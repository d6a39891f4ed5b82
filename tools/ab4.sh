#!/usr/bin/env bash
# A/B of two libpxr.so builds over the four BASELINE workloads, interleaved.
# usage: bash tools/ab4.sh <lib_a> <lib_b> [rounds]
a=$1; b=$2; n=${3:-2}
for i in $(seq "$n"); do
  for lib in "$a" "$b"; do
    for m in "Humanoid video" "HalfCheetah none" "Walker2d video" "Ant color"; do
      set -- $m
      echo -n "$(basename "$lib") "
      PXR_LIB_PATH=$lib python tools/prof_step.py --timed 50 --model "$1" --mode "$2" | tail -1
    done
  done
done
