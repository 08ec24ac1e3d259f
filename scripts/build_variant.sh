#!/bin/bash
# build_variant.sh NAME "-DFLAG=V ..." [source.cu] : libsubsurf_b200.so with one source
# (default sor_tma.cu) rebuilt under
# extra defines, written to variants/NAME.so (git-ignored; travels with gpurun).
# Select it with SUBSURF_B200_LIB=variants/NAME.so.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2111_11866_b200/csrc
make -s -C $C >/dev/null
mkdir -p $ROOT/variants/$1
ARCH="-gencode arch=compute_100a,code=sm_100a"
SRC=${3:-sor_tma.cu}
case $SRC in /*) ;; *) SRC=$C/$SRC ;; esac  # a path outside csrc/ replaces the same-named source
OBJ=$(basename ${SRC%.cu}).o
nvcc $ARCH -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-fvisibility=hidden -I$ROOT/include $2 \
    -I$C -c -o $ROOT/variants/$1/$OBJ $SRC
OBJS=$(ls $C/build/*.o | grep -v "/$OBJ")
nvcc $ARCH -shared -o $ROOT/variants/$1.so $OBJS $ROOT/variants/$1/$OBJ -Xlinker -z,defs -lcudart_static -lrt -lpthread -ldl
echo variants/$1.so
