#!/bin/bash
# usage: tools/var_tiers.sh lib1.so lib2.so ...  -> per-tier cost + c5 bench per library variant
for L in "$@"; do
  echo "== $L"
  SPHKV_LIB=$PWD/$L timeout 300 python tools/tier_cost.py 2>&1 | grep -v "^$" | cut -c1-80
  SPHKV_LIB=$PWD/$L timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-dense --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 | tok/s %.1f kernel_ms %.4f frac %.3f' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac']))"
done
