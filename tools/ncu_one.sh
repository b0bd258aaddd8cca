#!/bin/bash
# usage: tools/ncu_one.sh <tag> "<bench args>"  -> full ncu capture of the 3rd k_ada_decode launch
TAG=$1; A=$2
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ada_decode -s 2 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --config c5 --profile --steps 1 --no-dense $A > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_$TAG.log
