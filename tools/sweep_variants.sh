#!/bin/bash
# Build libmtgp_b200 variants of the v2 generation kernel (pipe-balance switches, register
# targets) into paper_1501_07701_b200/variants/ for tools/sweep.py. Run after the main build.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_1501_07701_b200/csrc
OUT=$ROOT/paper_1501_07701_b200/variants
mkdir -p $OUT
OBJS="$CS/build/mtgp_capi.o $CS/build/mtgp_v1.o $CS/build/mtgp_plan.o $CS/build/gf2.o"
build() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -I$ROOT/include -I$CS "$@" \
       -c $CS/mtgp_v2.cu -o $OUT/$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name.so $OBJS $OUT/$name.o -lpthread
  rm -f $OUT/$name.o
}
for v in "$@"; do
  IFS=: read name flags <<< "$v"
  build $name $flags &
done
wait
ls $OUT
