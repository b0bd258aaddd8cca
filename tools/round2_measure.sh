#!/bin/bash
# Round-2 measurement batch (1 GPU): default bench line, reference arm,
# binding-budget sweep, other configs, ncu launch list + full capture of c5.
OUT=gpurun_out/${TAG:-m}; mkdir -p $OUT
( time timeout 900 python bench.py ) > $OUT/bench_c5_default.json 2> $OUT/bench_c5_default.err
tail -1 $OUT/bench_c5_default.json | cut -c1-400
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ) > $OUT/bench_c5_reference.json 2> $OUT/bench_c5_reference.err
tail -1 $OUT/bench_c5_reference.json | cut -c1-300
for R in 0.40 0.50 0.60; do
  timeout 900 python bench.py --reduction $R --steps 50 --warmup 3 --no-cpu --no-appends > $OUT/bench_c5_red$R.json 2> $OUT/bench_c5_red$R.err
  echo "red $R rc=$?"
done
timeout 1500 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "c4 rc=$?"
timeout 1500 python bench.py --config c2 --no-dense --steps 20 --warmup 3 --no-cpu > $OUT/bench_c2.json 2> $OUT/bench_c2.err; echo "c2 rc=$?"
timeout 2000 python bench.py --config c3 --no-dense --steps 10 --warmup 3 --no-cpu --no-appends > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "c3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(ada|dense|lse)' \
  --csv --log-file $OUT/launches_c5.csv python bench.py --profile --steps 1 --no-parity > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ada_decode -s 2 -c 1 \
  -o $OUT/prof_c5 python bench.py --profile --steps 1 --no-dense --no-parity > $OUT/ncu_full.log 2>&1
echo "full rc=$?"
