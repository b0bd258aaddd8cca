#!/bin/bash
# tools/ab_args.sh <config> <timeout> "<args 1>" "<args 2>" ... : one bench line per argument set (shipped lib)
C=$1; TO=$2; shift 2
mkdir -p gpurun_out/aa
i=0
for A in "$@"; do
  i=$((i+1))
  timeout $TO python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-appends --no-dense $A > gpurun_out/aa/$C_$i.json 2> gpurun_out/aa/$C_$i.err
  echo "[$A] rc=$?"
  tail -1 gpurun_out/aa/$C_$i.json | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); pa=d.get('parity') or {}
  print('  ada %.1f tok/s %.4f ms frac %.3f | parity %s' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'], pa.get('max_out_rel')))
except Exception as e: print('  no line', e)"
done
