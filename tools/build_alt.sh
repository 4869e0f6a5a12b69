#!/bin/bash
# Build an A/B variant of libfvcuda.so with extra -D flags: bash tools/build_alt.sh <name> "-DFOO=1 -DBAR=2"
set -e
name=$1; shift
flags="$*"
mkdir -p build/alt_$name
for f in paper_2306_16541_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags -c $f -o build/alt_$name/$b.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static build/alt_$name/*.o -o alt_$name.so
echo built alt_$name.so
