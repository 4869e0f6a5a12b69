# A/B the inference stages: bash tools/ab_infer.sh <variant>...  (alt_<variant>.so at the repo root)
for v in "$@"; do cp alt_$v.so paper_2306_16541_b200/libfvcuda.so; timeout 300 python bench.py --steps 5 --warmup 3 --no-train --no-scene --skip-cpu-baseline > gpurun_out/st_$v.log 2>&1; python -c "
import json,sys
l=[x for x in open('gpurun_out/st_$v.log') if x.startswith('{')][-1]; d=json.loads(l); print('$v', round(d['frames_per_s'],2), round(d['stages_ms']['offset'],3), round(d['stages_ms']['radiance'],3), round(d['stages_ms']['march_warp'],3))"; done
