#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list, ncu full capture of the step kernel.
set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $OUT/gpu_tests.log
if [ "${SANITIZE:-0}" = "1" ]; then
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "paper_litmus or pool_sizes or staging or c4_subset or slot_limits" > $OUT/sanitizer.log 2>&1; echo "sanitizer rc=$?" >> $OUT/sanitizer.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python tools/profile_run.py > $OUT/launches.log 2>&1; echo "ncu list rc=$?" >> $OUT/launches.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light|step_overflow)_kernel" -s 384 -c 3 -o $OUT/prof_step python tools/profile_run.py > $OUT/prof.log 2>&1; echo "ncu full rc=$?" >> $OUT/prof.log
ls -la $OUT
