#!/bin/bash
# usage: tools/launch_list.sh <tag> <lib.so> <config> -> per-launch durations of one profile step
TAG=$1; L=$2; C=$3
SPHKV_LIB=$PWD/$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_ada' \
  --csv --log-file gpurun_out/ll_$TAG.csv python bench.py --config $C --profile --steps 1 --no-dense --no-parity > gpurun_out/ll_$TAG.log 2>&1
python - gpurun_out/ll_$TAG.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; data = rows[1:]
ki = h.index("Kernel Name"); vi = h.index("Metric Value")
vals = [(r[ki][:30], float(r[vi].replace(",", ""))) for r in data if "gpu__time_duration" in r]
print(len(vals), "launches; durations (us):", [round(v / 1e3, 1) for _, v in vals][:30])
PY
