#!/bin/bash
# Build libropeslr_b200.so with one translation unit replaced (other source
# file and/or extra nvcc flags) into paper_2605_20659_b200/_variants/<name>.so
# for kernel experiments; load it with ROPESLR_LIBRARY=<path>.
#   usage: build_variant.sh <name> <object-name> <source.cu> [nvcc flags...]
#   e.g.   build_variant.sh p12 attn_sm100 csrc/attn_sm100.cu -DROPESLR_POLY_NUM=1 -DROPESLR_POLY_DEN=2
set -e
name=$1; obj=$2; src=$3; shift 3
cd "$(dirname "$0")/../paper_2605_20659_b200"
python -c "import build; build.build()" >/dev/null
rm -rf _variants/$name && mkdir -p _variants/$name
cp _build/*.o _variants/$name/
nvcc -x cu -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I ../include -I csrc "$@" -c "$src" -o _variants/$name/$obj.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/$name.so _variants/$name/*.o -lcudart_static -lrt -ldl -lpthread
echo _variants/$name.so
