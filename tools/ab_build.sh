#!/bin/bash
# Build an A/B variant of the library with extra nvcc defines into tools/_ab/<name>.so
# (same ABI; select it with CW_LIB_PATH).   tools/ab_build.sh name -DFOO -DBAR=2
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/tools/_ab/$NAME
mkdir -p $OUT
cd $ROOT/paper_2505_00690_b200/csrc
for f in sample crowd robot routes sceneio; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -I $ROOT/include \
       -Xcompiler -fPIC "$@" -c $f.cu -o $OUT/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/tools/_ab/$NAME.so $OUT/*.o
echo $ROOT/tools/_ab/$NAME.so
