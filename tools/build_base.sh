#!/usr/bin/env bash
# Build build/ab/libpxr_base.so from the committed sources (HEAD, or the rev in $1) for A/B timing
# against the working tree's paper_2502_00021_b200/libpxr.so.
set -e
root=$(git rev-parse --show-toplevel)
tmp=$(mktemp -d)
git -C "$root" archive "${1:-HEAD}" paper_2502_00021_b200/csrc include | tar -x -C "$tmp"
mkdir -p "$root/build/ab"
cd "$tmp/paper_2502_00021_b200/csrc"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -fmad=false -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -shared \
  -o "$root/build/ab/libpxr_base.so" pxr_render.cu pxr_ops.cu pxr_physics.cu pxr_policy.cu
rm -rf "$tmp"
