#!/bin/bash
# build/lib_<name>.so with extra -D flags on one source (profiling aid)
# usage: scripts/build_variant.sh <name> <source-stem> -DFOO=1 ...
name=$1; stem=$2; shift 2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  "$@" -c paper_2511_00868_b200/csrc/$stem.cu -o build/v_$name.o || exit 1
objs=""
for src in paper_2511_00868_b200/csrc/*.cu; do
  s=$(basename $src .cu); [ "$s" = "$stem" ] || objs="$objs build/$s.o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/lib_$name.so $objs build/v_$name.o -lcudart
