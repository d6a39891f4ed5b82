#!/usr/bin/env bash
# Build libpxr variants with other geometry / raster warp splits of the
# pipelined render kernel (-DPXR_PIPE_GWARPS) into build/var/ (run here, then
# time them on the GPU box with tools/pipe_prof.py through PXR_LIB_PATH).
set -e
cd "$(dirname "$0")/../paper_2502_00021_b200/csrc"
mkdir -p ../../build/var
for g in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
    -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr -DPXR_PIPE_GWARPS=$g -shared \
    -o ../../build/var/libpxr_gw$g.so pxr_render.cu pxr_render_pipe.cu pxr_ops.cu pxr_physics.cu pxr_policy.cu
done
