#!/bin/bash
# usage: tools/bench_libs_cfg.sh <config> "<bench args>" lib1.so lib2.so ...
C=$1; A="$2"; shift; shift
for L in "$@"; do
  SPHKV_LIB=$PWD/$L timeout 900 python bench.py --config $C --steps 10 --warmup 3 --no-dense --no-cpu --no-parity --no-appends $A 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C $L $A', '| tok/s %.1f kernel_ms %.4f frac %.3f' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac']))"
done
