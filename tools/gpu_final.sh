#!/bin/bash
# End-of-session GPU evidence for the committed build: tests, smoke, bench c3/c4/c6,
# ncu launch list + full capture of c3, then the 10^6-trace c3 parity run and a
# 2*10^5-trace c6 parity run.
set -x
OUT=gpurun_out
bash tools/gpu_round.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py --config c4 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --config c6 > $OUT/bench_c6.json 2> $OUT/bench_c6.err
timeout 1500 python tests/run_parity_1m.py > $OUT/parity_1m.log 2>&1; echo "rc=$?" >> $OUT/parity_1m.log
timeout 600 python tests/run_parity_1m.py --config 6 --traces 200000 > $OUT/parity_c6.log 2>&1; echo "rc=$?" >> $OUT/parity_c6.log
ls -la $OUT
