#!/bin/bash
# tools/ab_env.sh <config> <timeout> "<env 1>" "<env 2>" ... : one bench line per environment setting (shipped lib)
C=$1; TO=$2; shift 2
mkdir -p gpurun_out/ae
i=0
for E in "$@"; do
  i=$((i+1))
  env $E timeout $TO python bench.py --config $C --steps 50 --warmup 3 --no-cpu --no-appends --no-dense > gpurun_out/ae/${C}_$i.json 2> gpurun_out/ae/${C}_$i.err
  echo "[$E] rc=$?"
  tail -1 gpurun_out/ae/${C}_$i.json | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); pa=d.get('parity') or {}
  print('  ada %.1f tok/s %.4f ms frac %.3f | parity %s' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'], pa.get('max_out_rel')))
except Exception as e: print('  no line', e)"
done
