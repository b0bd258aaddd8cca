#!/bin/bash
# HEAD check on one box: GPU tests, smoke, default c5 bench line, c4 line.
OUT=gpurun_out/${TAG:-h}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $OUT/pytest_gpu.log; tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c5_default.json 2> $OUT/bench_c5_default.err; echo "c5 rc=$?"
tail -1 $OUT/bench_c5_default.json | cut -c1-600
timeout 1200 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "c4 rc=$?"
tail -1 $OUT/bench_c4.json | cut -c1-400
