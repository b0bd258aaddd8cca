#!/bin/bash
# Round-end style check on one GPU: default bench (ours), reference arm, ncu launch list + full capture.
OUT=gpurun_out; TAG=${1:-r1}
mkdir -p $OUT
( time timeout 900 python bench.py ) > $OUT/bench_default_$TAG.json 2> $OUT/bench_default_$TAG.err
tail -1 $OUT/bench_default_$TAG.json | cut -c1-3000; grep real $OUT/bench_default_$TAG.err
( time timeout 900 python bench.py --impl reference --steps 3 --warmup 1 ) > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
tail -1 $OUT/bench_ref_$TAG.json | cut -c1-1500; grep real $OUT/bench_ref_$TAG.err; tail -3 $OUT/bench_ref_$TAG.err
bash tools/ncu_check.sh c5 $TAG > /dev/null 2>&1
echo ncu done
