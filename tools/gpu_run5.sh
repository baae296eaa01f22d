#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_c4.txt
for round in 1 2; do for lib in exp_libs/*.so; do
  RKC_LIB=$lib timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag $(basename $lib .so) >> $OUT/ab_c4.txt 2>&1
done; done
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > $OUT/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $OUT/gpu_tests.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 1200 python bench.py --config c4 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "bench c4 rc=$?" >> $OUT/bench_c4.err
RKC_BENCH_WATCHDOG=500 timeout 600 python bench.py --gpus 2 --steps 3 --no-cpu-baseline > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "bench n2 rc=$?" >> $OUT/bench_n2.err
ls -la $OUT
