#!/bin/bash
# build an experimental libcbx variant: $1 = name, $2 = source (default bandit.cu), rest = extra nvcc flags
set -e
cd "$(dirname "$0")/.."
name=$1; shift
src=bandit.cu
if [[ "$1" == *.cu ]]; then src=$1; shift; fi
extra=""
[ "$src" = bandit.cu ] && extra="-fmad=false"
mkdir -p build/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude $extra "$@" -c paper_2602_02827_b200/csrc/$src -o build/var_$name/${src%.cu}.o
objs=$(ls build/*.o | grep -v "/${src%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name/libcbx.so build/var_$name/${src%.cu}.o $objs -cudart=static
echo built build/var_$name/libcbx.so
