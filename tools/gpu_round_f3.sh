#!/bin/bash
# c3 round (tests, bench, ncu launch list + full capture) plus the c6 (f3) bench line and captures.
set -x
OUT=gpurun_out
bash tools/gpu_round.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py --config c6 > $OUT/bench_c6.json 2> $OUT/bench_c6.err; echo "bench c6 rc=$?" >> $OUT/bench_c6.err
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c6.csv python tools/profile_run.py --config 6 > $OUT/launches_c6.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light|step_overflow)_kernel" -s 384 -c 3 -o $OUT/prof_step_c6 python tools/profile_run.py --config 6 > $OUT/prof_c6.log 2>&1; echo "ncu c6 rc=$?" >> $OUT/prof_c6.log
ls -la $OUT
