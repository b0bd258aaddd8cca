#!/bin/bash
# tools/ab_mix.sh <config> <timeout> "ENV|ARGS" ... : one bench line per (environment, bench args) pair
C=$1; TO=$2; shift 2
mkdir -p gpurun_out/am
i=0
for EA in "$@"; do
  i=$((i+1)); E=${EA%%|*}; A=${EA#*|}
  env $E timeout $TO python bench.py --config $C --steps 50 --warmup 3 --no-cpu --no-appends --no-dense $A > gpurun_out/am/${C}_$i.json 2> gpurun_out/am/${C}_$i.err
  echo "[$E | $A] rc=$?"
  tail -1 gpurun_out/am/${C}_$i.json | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); pa=d.get('parity') or {}
  print('  ada %.1f tok/s %.4f ms frac %.3f | parity logits %s out %s' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'], pa.get('max_logit_rel'), pa.get('max_out_rel')))
except Exception as e: print('  no line', e)"
  tail -2 gpurun_out/am/${C}_$i.err | cut -c1-300
done
