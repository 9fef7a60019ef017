#!/bin/bash
# Build an A/B variant of the library: scripts/ab_build.sh OUT.so [SRC_DIR|-] [-DMACRO=...]
# SRC_DIR defaults to the package dir; the output goes under ab/ (git-ignored, travels with gpurun).
out=$1; src=${2:--}; shift 2
root="$(cd "$(dirname "$0")/.." && pwd)"
[ "$src" = "-" ] && src="$root/paper_2306_13493_b200"
mkdir -p "$root/ab"
cd "$src"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -O3 -shared \
  -I"$root/include" "$@" -o "$root/ab/$out" csrc/capi.cu csrc/ce_sample.cu csrc/mgpcg.cu csrc/level_setup.cu csrc/setup.cpp csrc/group.cpp -ldl -lpthread
