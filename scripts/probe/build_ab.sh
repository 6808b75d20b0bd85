#!/bin/bash
# Build an A/B variant of the library: NAME FILE.cu "EXTRA FLAGS" -> paper_2312_17649_b200/_lib_ab/NAME.so
# (the other objects from _build/; measurement only, SC_LIB_PATH selects it at run time).
set -e
NAME=$1; SRC=$2; FLAGS=$3
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
C=$ROOT/paper_2312_17649_b200/csrc; B=$ROOT/paper_2312_17649_b200/_build; O=$ROOT/paper_2312_17649_b200/_lib_ab
mkdir -p $O/obj_$NAME
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr \
  -cudart static -Xptxas -v $FLAGS -c $C/$SRC -o $O/obj_$NAME/${SRC%.cu}.o 2> $O/obj_$NAME/ptxas.log
OBJS=""
for o in $B/*.o; do b=$(basename $o); [ "$b" == "${SRC%.cu}.o" ] && OBJS="$OBJS $O/obj_$NAME/$b" || OBJS="$OBJS $o"; done
nvcc $ARCH -shared -cudart static -Xcompiler -fPIC $OBJS -o $O/$NAME.so
echo built $O/$NAME.so
