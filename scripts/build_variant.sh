#!/bin/bash
# Build-time A/B variants of the walk kernels: compiles walk.cu with extra
# defines into paper_2010_04895_b200/libmhw_<name>.so (the other objects are
# those of the default build); load it with MHW_LIB=<path>.
#   bash scripts/build_variant.sh hashef -DMHW_HASH_HINT=1
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
PKG=paper_2010_04895_b200
[ -f $PKG/_obj/api.o ] || python -m $PKG.build > /dev/null
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
$NVCC -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-O2,-fvisibility=hidden -Xptxas -O3 -I include "$@" -c $PKG/csrc/walk.cu -o $PKG/_obj/walk_$NAME.o 2> /dev/null
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -o $PKG/libmhw_$NAME.so $PKG/_obj/graph.o $PKG/_obj/walk_$NAME.o \
  $PKG/_obj/exact.o $PKG/_obj/corpus.o $PKG/_obj/loader.o $PKG/_obj/api.o \
  -Xlinker --version-script=$PKG/_obj/exports.map -lpthread
echo built $PKG/libmhw_$NAME.so "$@"
