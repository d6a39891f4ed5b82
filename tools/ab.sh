#!/usr/bin/env bash
# A/B timing of two libpxr.so builds on the same box, interleaved.
# usage: bash tools/ab.sh <lib_a> <lib_b> [prof_step args...]
a=$1; b=$2; shift 2
for i in 1 2 3; do
  for lib in "$a" "$b"; do
    echo -n "$(basename $lib): "
    PXR_LIB_PATH=$lib python tools/prof_step.py --timed 50 "$@" 2>&1 | tail -1
  done
done
