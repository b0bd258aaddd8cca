#!/bin/bash
# usage: tools/var_args.sh <config> "<args1>" "<args2>" ... -> bench line per argument set
C=$1; shift
for A in "$@"; do
  timeout 400 python bench.py --config $C --steps 30 --warmup 5 --no-cpu --no-dense --no-parity $A 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C [$A]', '| tok/s %.1f kern %.4f frac %.3f' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac']))"
done
