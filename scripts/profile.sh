#!/bin/bash
# Profiling pass for a gpurun box (1 GPU).  Each ncu run follows the same command
# run plainly (exit 0) first, per /opt/skills/guides/B200_PROFILING.md.
#   bash scripts/profile.sh [workload] [update]
set -u
W=${1:-mesh}
U=${2:-jacobi}
OUT=gpurun_out
CMD="python bench.py --workload $W --update $U --iters 20 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-alt"
mkdir -p $OUT
# 1) launch list: every launch of one reduced step with its device time
$CMD > $OUT/plain_${W}_${U}.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${W}_${U}.csv $CMD > $OUT/ncu_launches_${W}_${U}.log 2>&1
echo "launch list rc=$?"
# 2) full capture of the dominant kernel (first level-0 launch of the timed step)
K=layout_iter; S=60; C=1
# sampled (split form), 20 iterations per level: coarse levels 1 draw + 20 applies
# each, level 0 (256 MB draw chunks = 5 epochs) 4 draws + 20 applies -> 87 matching
# launches per step; the timed step's level 0 starts at launch 87 + 63 = 150 with
# draw(chunk 0), draw(chunk 1), apply(epoch 0)
# (level 0 of the mesh runs apply_snap_kernel after a snap_copy_kernel per epoch)
# and draws only the pairs in the draw pass (8-byte records: 18 epochs per chunk, two
# draw launches for 20 epochs): 3 x 21 + 22 = 85 matching launches per step, the timed
# step's level 0 from launch 148 -- captured from 146: two coarse applies, the two
# draw launches, the first two level-0 epochs
[ "$U" = "sampled" ] && K="draw_kernel|apply_kernel|apply_snap_kernel|apply_negsnap_kernel" && S=146 && C=6
$CMD > $OUT/plain2_${W}_${U}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s $S -c $C -f \
      -o $OUT/full_${W}_${U} $CMD > $OUT/ncu_full_${W}_${U}.log 2>&1
echo "full capture rc=$?"
# 3) the per-epoch snapshot refresh of the sampled form
if [ "$U" = "sampled" ]; then
  ncu --set full --clock-control none -k "regex:snap_copy_kernel|negsnap_refresh_kernel" -s 30 -c 1 -f \
      -o $OUT/full_${W}_${U}_snapcopy $CMD > $OUT/ncu_full_${W}_${U}_snapcopy.log 2>&1
  echo "snap copy capture rc=$?"
fi
