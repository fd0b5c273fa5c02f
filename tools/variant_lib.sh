#!/bin/bash
# Build an experiment variant of libstmg_b200.so with one translation unit
# recompiled under extra -D switches:
#   tools/variant_lib.sh <name> <source.cu> [-DFOO=1 ...]
# -> paper_2502_09159_b200/_build/variants/<name>.so (load with STMG_LIB=...)
set -e
name=$1; src=$2; shift 2
B=paper_2502_09159_b200/_build; V=$B/variants; mkdir -p $V
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 -ccbin /usr/bin/g++ "$@" \
  -c paper_2502_09159_b200/csrc/$src -o $V/$name.$src.o
objs=$(ls $B/*.o | grep -v "/$src.o$")
nvcc $ARCH -ccbin /usr/bin/g++ -shared -o $V/$name.so $objs $V/$name.$src.o -lcudart -ldl
echo $V/$name.so
