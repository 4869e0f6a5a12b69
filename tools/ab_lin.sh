#!/bin/bash
# A/B the training layer GEMMs (tools/time_lin.py) for alt_<variant>.so builds
cp paper_2306_16541_b200/libfvcuda.so /tmp/keep.so
for v in "$@"; do cp alt_$v.so paper_2306_16541_b200/libfvcuda.so; echo "== $v"; timeout 200 python tools/time_lin.py 2>&1 | head -3; done
cp /tmp/keep.so paper_2306_16541_b200/libfvcuda.so
