#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of the prefill kernel.
set -x
OUT=gpurun_out
TAG=${1:-r}
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > $OUT/pytest_$TAG.log 2>&1; tail -5 $OUT/pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; tail -3 $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; tail -c 3000 $OUT/bench_$TAG.json; tail -5 $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --decode-steps 64 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 2 -c 1 \
    -o $OUT/prof_tc_$TAG python tools/prof_driver.py > $OUT/ncu_full_$TAG.log 2>&1
tail -3 $OUT/ncu_full_$TAG.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_step -s 5 -c 1 \
    -o $OUT/prof_dec_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --decode-steps 64 > $OUT/ncu_dec_$TAG.log 2>&1
tail -3 $OUT/ncu_dec_$TAG.log
ls -la $OUT
