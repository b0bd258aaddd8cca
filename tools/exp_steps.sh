#!/bin/bash
# decode-only and full decode step (gate + appends) per library: tools/exp_steps.sh <config> lib...
C=$1; shift
for L in "$@"; do
  SPHKV_LIB=$PWD/$L timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu --no-dense --no-parity $EXTRA 2>/dev/null | tail -1 | \
    python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d.get('decode_step_with_appends') or {}
print('$C $(basename $L) $EXTRA | decode %.1f tok/s | step with appends %s tok/s (%s ms)' % (d['value'], a.get('value'), a.get('ms_per_step')))"
done
