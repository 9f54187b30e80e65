#!/bin/bash
# Build an alternative libctk_b200.so with extra nvcc flags for kernel A/B timing:
#   tools/build_variant.sh NAME -DSOME_MACRO ...   ->  build_variants/NAME/libctk_b200.so
# (load it with CTK_B200_LIB=build_variants/NAME/libctk_b200.so)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
D=$ROOT/build_variants/$NAME
mkdir -p $D
make -s -C $ROOT/paper_2211_14212_b200/csrc -j8 OBJ=$D/obj OUT=$D \
  NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fno-fast-math -Xptxas -v $*"
ls -la $D/libctk_b200.so
