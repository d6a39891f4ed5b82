#!/usr/bin/env bash
# A/B of render CTA sizes: libpxr_<threads>.so built with -DPXR_RENDER_THREADS=<threads> into build/var/
# (nvcc flags as csrc/Makefile); usage: bash tools/ab_threads.sh
for i in 1 2; do
for t in 768 640 704 832; do
  for m in "Humanoid video" "HalfCheetah none" "Walker2d video" "Ant color"; do
    set -- $m
    echo -n "$t $1 "
    PXR_LIB_PATH=build/var/libpxr_$t.so timeout 120 python tools/prof_step.py --timed 50 --model "$1" --mode "$2" 2>&1 | tail -1
  done
done; done
