#!/bin/bash
# A/B timing of librkc variants on c4 (10k traces x 65536 blocks), 64 steps.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_c4.txt
for lib in exp_libs/*.so; do
  RKC_LIB=$lib timeout 300 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --steps ${C4_STEPS:-64} --reps 2 --tag $(basename $lib .so) >> $OUT/ab_c4.txt 2>&1
done
cat $OUT/ab_c4.txt
