#!/bin/bash
# build an experimental libcbx variant: $1 = name, rest = extra nvcc flags for bandit.cu
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude -fmad=false "$@" -c paper_2602_02827_b200/csrc/bandit.cu -o build/var_$name/bandit.o
objs=$(ls build/*.o | grep -v "/bandit.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name/libcbx.so build/var_$name/bandit.o $objs -cudart=static
echo built build/var_$name/libcbx.so
