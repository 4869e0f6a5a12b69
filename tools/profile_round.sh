#!/bin/bash
# Evidence capture for profiles/ (run on the GPU box from the repo root):
#   bench line, launch lists (bench + training), --set full of the C2 kernels, the sparse
#   (opaque-subject + occupancy) march, the gather probe and the training kernels.
#   Usage: bash tools/profile_round.sh <tag>
tag=${1:-r02}
o=gpurun_out
timeout 900 python bench.py > $o/bench_$tag.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $o/bench_launches_$tag.csv \
  python bench.py --steps 2 --warmup 3 --skip-cpu-baseline --no-occ-variants --no-trained > $o/bench_ncu_$tag.log 2>&1; echo "launch list rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/train_launches_$tag.csv \
  python tools/time_train.py 2 > $o/train_ncu_$tag.log 2>&1; echo "train launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_march_warp|k_offset_tc|k_radiance_tc|k_radiance_ws" \
  -s 3 -c 3 -o $o/infer_$tag -f python tools/time_stages.py --reps 2 > $o/infer_ncu_$tag.log 2>&1; echo "infer full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_march_warp" -s 1 -c 1 \
  -o $o/march_opaque_$tag -f python tools/time_stages.py --opaque --reps 2 > $o/march_opaque_ncu_$tag.log 2>&1; echo "sparse march rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"k_gather_probe" -c 2 -o $o/gather_$tag -f \
  python tools/gather_probe.py > $o/gather_ncu_$tag.log 2>&1; echo "gather probe rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_rows|k_dw|k_hash_bwd|k_warp_bwd|k_hash_fwd|k_narrow_dx|k_adam_update" -c 30 -o $o/train_$tag -f \
  python tools/time_train.py 1 > $o/train_full_ncu_$tag.log 2>&1; echo "train full rc=$?"
# summaries on the box (gpurun copies back <= 64 MiB): tables + key metrics, then drop big reports
for r in infer march_opaque gather train; do
  f=$o/${r}_$tag.ncu-rep
  [ -f $f ] || continue
  python tools/ncu_table.py $f "$r $tag" > $o/${r}_${tag}_table.txt 2>&1
  python tools/ncu_summary.py $f > $o/${r}_${tag}_summary.txt 2>&1
  sz=$(stat -c %s $f); if [ $sz -gt 12000000 ]; then rm -f $f; echo "dropped $f ($sz bytes)"; fi
done
python tools/launch_summary.py $o/bench_launches_$tag.csv > $o/bench_launches_${tag}_summary.txt 2>&1
python tools/launch_summary.py $o/train_launches_$tag.csv > $o/train_launches_${tag}_summary.txt 2>&1
du -sh $o
