#!/bin/bash
# Build an experiment variant of libstmg_b200.so with some translation units
# recompiled under extra -D switches:
#   tools/variant_lib.sh <name> "<src1.cu src2.cu ...>" [-DFOO=1 ...]
# -> paper_2502_09159_b200/_build/variants/<name>.so (load with STMG_LIB=...)
set -e
name=$1; srcs=$2; shift 2
B=paper_2502_09159_b200/_build; V=$B/variants; mkdir -p $V
ARCH="-gencode arch=compute_100a,code=sm_100a"
objs=$(ls $B/*.o)
pids=()
for src in $srcs; do
  nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O3 -ccbin /usr/bin/g++ -I include "$@" \
    -c paper_2502_09159_b200/csrc/$src -o $V/$name.$src.o &
  pids+=($!)
  objs=$(echo "$objs" | grep -v "/$src.o$")
done
for p in "${pids[@]}"; do wait $p; done
nvcc $ARCH -ccbin /usr/bin/g++ -shared -o $V/$name.so $objs $(for src in $srcs; do echo $V/$name.$src.o; done) -lcudart -ldl
echo $V/$name.so
