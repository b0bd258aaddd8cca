#!/bin/bash
# Bench lines for several configs on one GPU: tools/bench_cfgs.sh <tag> "<cfg args>" ...
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
i=0
for A in "$@"; do
  i=$((i+1))
  timeout 1500 python bench.py $A > $OUT/bench_${TAG}_$i.json 2> $OUT/bench_${TAG}_$i.err
  echo "== $A rc=$?"
  python - $OUT/bench_${TAG}_$i.json $OUT/bench_${TAG}_$i.err <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    dn = d.get("dense_baseline") or {}
    pa = d.get("parity") or {}
    print("tok/s %.1f e2e %.1f kern %.4f frac %.3f | dense %.1f (%.3f) x%.3f | parity lg %.2e out %.2e | kv/tok %.0f res %.3f str %s" % (
        d["value"], d["e2e"]["value"], d["roofline"]["kernel_ms_per_launch"], d["roofline"]["frac"],
        dn.get("value", 0), dn.get("frac_of_peak", 0), d.get("speedup_vs_dense") or 0,
        pa.get("max_logit_rel", -1), pa.get("max_out_rel", -1), d["kv_bytes_per_token"],
        d["resident_ratio_vs_dense"], d.get("streamed_ratio_vs_dense")))
    print("tiers", d["budget"]["tier_items"])
except Exception as e:
    print("FAILED", e, open(sys.argv[2]).read()[-1500:])
PY
done
