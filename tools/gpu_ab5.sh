#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab.txt
for round in 1 2; do
  for lib in exp_libs/*.so; do
    RKC_LIB=$lib timeout 300 python tools/step_timing.py --tag c3_$(basename $lib .so) >> $OUT/ab.txt 2>&1
    RKC_LIB=$lib timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$(basename $lib .so) >> $OUT/ab.txt 2>&1
  done
done
cat $OUT/ab.txt
