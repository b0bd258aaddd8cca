#!/bin/bash
# usage: tools/build_variant.sh <name> "<-D flags>"  -> variants/lib<name>.so (GP=2 only unless flags override)
set -e
cd "$(dirname "$0")/.."
mkdir -p variants build/var_$1
A="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr --extended-lambda"
C=paper_2605_18856_b200/csrc
OBJ=build/obj
nvcc $A $2 -c ${SRC:-$C/decode.cu} -o build/var_$1/decode.o -Xptxas -v 2> build/var_$1/ptxas.log
nvcc $A -shared -o variants/lib$1.so build/var_$1/decode.o $(ls $OBJ/*.o | grep -v decode.o) -lcudart
grep -A1 "k_ada_decode" build/var_$1/ptxas.log | grep "registers\|spill" | head -2
