#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh NAME "-DFLAG=..." -> build/var/NAME.so
set -e
NAME=$1; shift
mkdir -p build/var/$NAME
for f in paper_2501_02573_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
       -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -c $f -o build/var/$NAME/$b.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/var/$NAME.so build/var/$NAME/*.o
echo built build/var/$NAME.so
