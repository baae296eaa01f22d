#!/bin/bash
# Session-3 A/B #14: grid-pacing margin (1/32, 1/16, 1/64 of the traces; max of the last 4 counts),
# then the 2-rank debug.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3n.txt
for lib in q4_nopace q0_pace q1_pace16 q2_pacemax q3_pace64; do
  RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3n.txt 2>&1
  for c in 3 6 8; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --config $c --tag c${c}_$lib >> $OUT/ab_s3n.txt 2>&1
  done
done
cat $OUT/ab_s3n.txt
bash tools/gpu_debug_n2.sh
