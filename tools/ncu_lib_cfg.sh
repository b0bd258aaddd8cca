#!/bin/bash
# usage: tools/ncu_lib_cfg.sh <tag> <lib.so> <config> <skip> -> full ncu of one k_ada_decode launch
TAG=$1; L=$2; C=$3; S=${4:-2}
SPHKV_LIB=$PWD/$L timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ada_decode -s $S -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --config $C --profile --steps 1 --no-dense --no-parity > gpurun_out/ncu_$TAG.log 2>&1
echo "$TAG rc=$?"
