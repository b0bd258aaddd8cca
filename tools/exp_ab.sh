#!/bin/bash
# A/B on one box: tools/exp_ab.sh <config> "<bench args>" lib1 lib2 ...  (prints ADA + dense per lib)
C=$1; A="$2"; shift; shift
for L in "$@"; do
  SPHKV_LIB=$PWD/$L timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-appends $A 2>/dev/null | tail -1 | \
    python -c "
import json,sys; d=json.loads(sys.stdin.read()); dn=d.get('dense_baseline') or {}
pa=d.get('parity') or {}
print('$C $(basename $L) $A | ada %.1f tok/s %.4f ms frac %.3f | dense %s frac %s | parity %s' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'], dn.get('value'), dn.get('frac_of_peak'), pa.get('max_out_rel')))"
done
