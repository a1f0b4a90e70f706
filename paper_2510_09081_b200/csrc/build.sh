#!/bin/bash
# Builds liblvx_b200.so (sm_100a only) next to the Python package.  -fmad=false: no FMA
# contraction anywhere, the integer outputs must match the f64 CPU reference bit for bit.
set -e
cd "$(dirname "$0")"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
OUT=${LVX_OUT:-../liblvx_b200.so}
$NVCC -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 \
      -Xcompiler -fPIC -shared ${LVX_NVCC_EXTRA} \
      upload.cu voxelize.cu cull.cu abuffer.cu bricks.cu shade.cu render.cu -o $OUT
echo "built $(realpath $OUT)"
