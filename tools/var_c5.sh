#!/bin/bash
# usage: tools/var_c5.sh lib1.so ... -> c5 bench line per library variant (+ tier 1/5 cost)
for L in "$@"; do
  SPHKV_LIB=$PWD/$L timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-dense 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', '| tok/s %.1f kern %.4f frac %.3f' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac']))"
done
