#!/bin/bash
# tools/ab1.sh <config> <timeout> "<bench args>" lib ... : one bench line per lib into gpurun_out/ab/
C=$1; TO=$2; A="$3"; shift 3
mkdir -p gpurun_out/ab
for L in "$@"; do
  N=$(basename $L .so)_$C
  ( time SPHKV_LIB=$PWD/$L timeout $TO python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-appends $A ) > gpurun_out/ab/$N.json 2> gpurun_out/ab/$N.err
  echo "$N rc=$?"
  tail -1 gpurun_out/ab/$N.json | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); dn=d.get('dense_baseline') or {}; pa=d.get('parity') or {}
  print('  ada %.1f tok/s %.4f ms frac %.3f | dense %s frac %s | parity %s' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'], dn.get('value'), dn.get('frac_of_peak'), pa.get('max_out_rel')))
except Exception as e: print('  no line', e)"
  tail -3 gpurun_out/ab/$N.err
done
