#!/bin/bash
# ncu evidence for the bench's dominant kernels (1 GPU).
# usage: tools/ncu_check.sh [config] [tag] [kernel regex for --set full]
CFG=${1:-c5}
TAG=${2:-r1}
K=${3:-k_ada_decode}
OUT=gpurun_out
mkdir -p $OUT
# launch list of one profile step (32 ADA + 32 merge + 32 dense + 32 merge launches)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(ada|dense|lse)' \
  --csv --log-file $OUT/launches_${CFG}_$TAG.csv python bench.py --config $CFG --profile --steps 1 \
  > $OUT/ncu_launch_${CFG}_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 2 -c 1 \
  -o $OUT/prof_${CFG}_$TAG python bench.py --config $CFG --profile --steps 1 --no-dense \
  > $OUT/ncu_full_${CFG}_$TAG.log 2>&1
echo "full rc=$?"
tail -3 $OUT/ncu_full_${CFG}_$TAG.log
