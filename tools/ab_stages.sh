#!/bin/bash
# A/B stage times of alt_<variant>.so builds: bash tools/ab_stages.sh "<time_stages args>" v1 v2 ...
args=$1; shift
cp paper_2306_16541_b200/libfvcuda.so /tmp/libfvcuda.keep.so
for v in "$@"; do
  cp alt_$v.so paper_2306_16541_b200/libfvcuda.so
  echo "$v: $(timeout 300 python tools/time_stages.py $args 2>&1 | tail -1)"
done
cp /tmp/libfvcuda.keep.so paper_2306_16541_b200/libfvcuda.so
