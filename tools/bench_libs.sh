#!/bin/bash
# usage: tools/bench_libs.sh "<bench args>" lib1.so lib2.so ...
A="$1"; shift
for L in "$@"; do
  SPHKV_LIB=$PWD/$L python tools/debug_tiers.py 2>&1 | grep "max logit" | awk '{m=($NF>m)?$NF:m} END {printf "max tier err %s  ", m}'
  SPHKV_LIB=$PWD/$L python bench.py --config c5 --steps 10 --warmup 3 --no-dense --no-cpu --no-parity --no-appends $A 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L $A', '| tok/s %.1f kernel_ms %.4f frac %.3f' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac']))"
done
