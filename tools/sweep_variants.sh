#!/bin/bash
# Build libmtgp_b200 variants of the generation kernels (pipe-balance switches, register
# targets) into paper_1501_07701_b200/variants/ for tools/sweep.py. Run after the main build.
#   tools/sweep_variants.sh "name:-DFLAG=1 -DOTHER=2" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
CS=$ROOT/paper_1501_07701_b200/csrc
OUT=$ROOT/paper_1501_07701_b200/variants
mkdir -p $OUT
OBJS=$(ls $CS/build/*.o)
NV="nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -I$ROOT/include -I$CS"
# VARIANT_SRCS (default: the v2 + v3 kernels) are rebuilt with the variant's flags and replace
# their objects from the main build.
VARIANT_SRCS=${VARIANT_SRCS:-"mtgp_v2 mtgp_v3"}
build() {
  name=$1; shift
  objs=""
  for f in $OBJS; do
    b=$(basename $f .o)
    case " $VARIANT_SRCS " in *" $b "*) ;; *) objs="$objs $f";; esac
  done
  for v in $VARIANT_SRCS; do
    $NV "$@" -c $CS/$v.cu -o $OUT/$name.$v.o
    objs="$objs $OUT/$name.$v.o"
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/$name.so $objs -lpthread
  for v in $VARIANT_SRCS; do rm -f $OUT/$name.$v.o; done
}
for v in "$@"; do
  IFS=: read name flags <<< "$v"
  build $name $flags &
done
wait
ls $OUT
