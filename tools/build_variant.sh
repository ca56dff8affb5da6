#!/bin/bash
# Build libvpipe_b200.so with extra compile-time flags into build_variants/<name>/
# (developer A/B: VPIPE_LIB=build_variants/<name>/libvpipe_b200.so python bench.py ...)
#   tools/build_variant.sh f32early -DVP_F32_EARLY=1
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build_variants/$name
mkdir -p "$out"
make -C "$root/paper_2411_05288_b200/csrc" -j4 OUT="$out" \
  NVFLAGS="-std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -Wall -I../../include $*"
echo "$out/libvpipe_b200.so"
