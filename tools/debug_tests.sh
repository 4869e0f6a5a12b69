#!/bin/bash
# Bounds-checked build (-DFV_DEBUG=1: FV_ASSERT traps on out-of-range gather / staging
# indices) run through the GPU tests, smoke() and the every-kernel smoke -- the stand-in for
# compute-sanitizer, which is closed on the GPU pool.  On the GPU box: bash tools/debug_tests.sh
set -e
[ -f alt_dbg.so ] || bash tools/build_alt.sh dbg -DFV_DEBUG=1
cp paper_2306_16541_b200/libfvcuda.so /tmp/libfvcuda.keep.so
cp alt_dbg.so paper_2306_16541_b200/libfvcuda.so
trap 'cp /tmp/libfvcuda.keep.so paper_2306_16541_b200/libfvcuda.so' EXIT
python -m pytest tests -q -m gpu -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/sanitize_smoke.py 2>&1 | tail -1
