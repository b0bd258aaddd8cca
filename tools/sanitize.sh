#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py: memcheck, racecheck, synccheck, initcheck
OUT=gpurun_out/sanitize
mkdir -p $OUT
python tools/sanitize_cases.py > $OUT/plain.log 2>&1; tail -1 $OUT/plain.log
for T in ${TOOLS:-memcheck synccheck racecheck}; do
  timeout 1500 compute-sanitizer --tool $T --target-processes all --kernel-name kns=sphkv \
    python tools/sanitize_cases.py > $OUT/$T.log 2>&1
  echo "$T rc=$? $(grep -c 'ERROR SUMMARY\|========= ' $OUT/$T.log) lines; $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY\|sanitize cases' $OUT/$T.log | tr '\n' ' ')"
done
