#!/bin/bash
# One GPU iteration: parity tests, per-tier debug, bench option sweep.
# usage: tools/gpu_iter.sh <tag> "<bench args 1>" "<bench args 2>" ...
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python tools/debug_tiers.py > $OUT/tiers_$TAG.log 2>&1; grep "max logit" $OUT/tiers_$TAG.log | awk '{print $1,$2,$3,$NF}' | tr '\n' ';'; echo
for A in "$@"; do
  timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu $A > $OUT/b.json 2> $OUT/b.err
  python - "$A" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
    dn = d.get("dense_baseline") or {}
    print(sys.argv[1], "| tok/s %.1f kern %.4f frac %.3f | dense %.1f | x%.3f | tiers %s" % (
        d["value"], d["roofline"]["kernel_ms_per_launch"], d["roofline"]["frac"],
        dn.get("value", 0), d.get("speedup_vs_dense") or 0, d["budget"].get("tier_items")))
except Exception as e:
    print(sys.argv[1], "FAILED", e, open("gpurun_out/b.err").read()[-800:])
PY
done
