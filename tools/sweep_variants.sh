#!/bin/bash
# Build libmtgp_b200 variants of the generation kernels (pipe-balance switches, register
# targets) into paper_1501_07701_b200/variants/ for tools/sweep.py. Run after the main build.
#   tools/sweep_variants.sh "name:-DFLAG=1 -DOTHER=2" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_1501_07701_b200/csrc
OUT=$ROOT/paper_1501_07701_b200/variants
mkdir -p $OUT
OBJS="$CS/build/mtgp_capi.o $CS/build/mtgp_v1.o $CS/build/mtgp_plan.o $CS/build/mtgp_mt.o $CS/build/mtgp_stat.o $CS/build/gf2.o $CS/build/sha1.o $CS/build/stat_host.o"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -I$ROOT/include -I$CS"
build() {
  name=$1; shift
  $NV "$@" -c $CS/mtgp_v2.cu -o $OUT/$name.v2.o
  $NV "$@" -c $CS/mtgp_v3.cu -o $OUT/$name.v3.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name.so $OBJS $OUT/$name.v2.o $OUT/$name.v3.o -lpthread
  rm -f $OUT/$name.v2.o $OUT/$name.v3.o
}
for v in "$@"; do
  IFS=: read name flags <<< "$v"
  build $name $flags &
done
wait
ls $OUT
