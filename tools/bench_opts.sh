#!/bin/bash
# usage: tools/bench_opts.sh "<bench args>" ["<bench args>" ...]  -> one summary line per option set
for A in "$@"; do
  python bench.py --config c5 --steps 10 --warmup 3 --no-dense --no-cpu $A 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$A', '| tok/s %.1f kernel_ms %.4f frac %.3f' % (d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac']))"
done
