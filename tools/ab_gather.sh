#!/bin/bash
# A/B of the gather probe (real stream / random points) for alt_<variant>.so builds
cp paper_2306_16541_b200/libfvcuda.so /tmp/libfvcuda.keep.so
for v in "$@"; do
  cp alt_$v.so paper_2306_16541_b200/libfvcuda.so
  echo "$v: $(timeout 300 python -c "
import sys, torch; sys.path.insert(0, '.')
import bench
from paper_2306_16541_b200 import scene as psc
from paper_2306_16541_b200.model import FreeviewModel
from paper_2306_16541_b200.render import RenderSettings, Renderer
sc = psc.make_scene(psc.config('c2')); nets = FreeviewModel(sc)
st = RenderSettings.from_config(sc.cfg, seed=sc.jitter_seed)
r = bench.gather_rates(nets, Renderer(), sc.camera, st, torch.device('cuda'), reps=5)
print('real %.3f ms  random %.3f ms' % (r['real_stream']['ms'], r['random_points']['ms']))
" 2>&1 | tail -1)"
done
cp /tmp/libfvcuda.keep.so paper_2306_16541_b200/libfvcuda.so
