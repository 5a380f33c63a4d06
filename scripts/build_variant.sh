#!/bin/bash
# Build an A/B variant of the library: scripts/build_variant.sh NAME -DFLAG=1 ...
# -> build/variants/NAME.so (select with TREEATTN_B200_LIB=build/variants/NAME.so)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variants/$name; mkdir -p $out
C=paper_2404_00242_b200/csrc
objs=""
for f in $C/*.cu; do o=$out/$(basename $f).o; /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC -Iinclude -I$C "$@" -c $f -o $o & objs="$objs $o"; done
for f in $C/*.cpp; do o=$out/$(basename $f).o; g++ -O3 -std=c++20 -fPIC -Iinclude -I$C -I/usr/local/cuda/include "$@" -c $f -o $o & objs="$objs $o"; done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/$name.so $objs -cudart shared
echo build/variants/$name.so
