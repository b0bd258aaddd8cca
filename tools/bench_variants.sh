#!/bin/bash
# usage: tools/bench_variants.sh lib1.so lib2.so ...   (debug: per-variant parity + c5 timing)
for L in "$@"; do
  echo "== $L"
  SPHKV_LIB=$PWD/$L python tools/debug_tiers.py 2>&1 | grep "max logit" | awk '{print $2, $3, $5, $8}' | tr '\n' ' '; echo
  SPHKV_LIB=$PWD/$L timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-dense --no-cpu --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('tok/s %.1f  kernel_ms %.4f  GB/s %.0f frac %.3f' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['achieved'], d['roofline']['frac']))"
done
