#!/bin/bash
# build an experimental libcbx variant: $1 = name, $2 = source (default: the bandit units bandit*.cu), rest = extra
# nvcc flags; the other objects come from the default build in build/
set -e
cd "$(dirname "$0")/.."
name=$1; shift
srcs=$(cd paper_2602_02827_b200/csrc && ls bandit*.cu | tr "\n" " ")
if [[ "$1" == *.cu ]]; then srcs=$1; shift; fi
mkdir -p build/var_$name
pids=""
for src in $srcs; do
  extra=""
  [[ $src == bandit* ]] && extra="-fmad=false"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude $extra "$@" -c paper_2602_02827_b200/csrc/$src -o build/var_$name/${src%.cu}.o &
  pids="$pids $!"
done
for p in $pids; do wait $p; done
objs=""
for o in build/*.o; do b=$(basename $o); [ -f build/var_$name/$b ] || objs="$objs $o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var_$name/libcbx.so build/var_$name/*.o $objs -cudart=static
echo built build/var_$name/libcbx.so
