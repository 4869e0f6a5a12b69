# A/B the training scatter kernels: bash tools/ab_train.sh <variant>...  (alt_<variant>.so at the repo root)
for v in "$@"; do cp alt_$v.so paper_2306_16541_b200/libfvcuda.so; echo "== $v"; timeout 200 python tools/time_hash_bwd.py 2>&1 | tail -2; timeout 200 python tools/time_warp_bwd.py 2>&1 | tail -1; done
