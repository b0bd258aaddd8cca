#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full capture.
# usage: tools/gpu_check.sh [config] [tag]
CFG=${1:-c5}
TAG=${2:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > $OUT/pytest_gpu_$TAG.log
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; tail -1 $OUT/smoke_$TAG.log
timeout 1200 python bench.py --config $CFG --steps 20 --warmup 5 > $OUT/bench_${CFG}_$TAG.log 2>&1
tail -1 $OUT/bench_${CFG}_$TAG.log | cut -c1-1500
