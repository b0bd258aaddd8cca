#!/bin/bash
# usage: tools/ncu_lib.sh <tag> <lib.so> ["<bench args>"] -> full ncu capture of the 3rd k_ada_decode launch
TAG=$1; L=$2; A=$3
SPHKV_LIB=$PWD/$L timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ada_decode -s 2 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --config c5 --profile --steps 1 --no-dense --no-parity $A > gpurun_out/ncu_$TAG.log 2>&1
echo "$TAG rc=$?"
