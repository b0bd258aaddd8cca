#!/bin/bash
# usage: tools/var_cfg.sh <config> lib1.so ... -> bench line per library variant for one config
C=$1; shift
for L in "$@"; do
  SPHKV_LIB=$PWD/$L timeout 400 python bench.py --config $C --steps 30 --warmup 5 --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C $L', '| tok/s %.1f kern %.4f frac %.3f dense %s' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'], (d.get('dense_baseline') or {}).get('value')))"
done
