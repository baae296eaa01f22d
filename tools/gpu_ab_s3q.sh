#!/bin/bash
# Session-3 A/B #17: overflow grid of 296 CTAs when the step grid is paced (+ rank select).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3q.txt
RKC_LIB=exp_libs/t2_ovf296_rs.so timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/par_t2.log 2>&1; echo "rc=$?" >> $OUT/par_t2.log
for round in 1 2; do
  for lib in t0_head t1_ovf296 t2_ovf296_rs; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3q.txt 2>&1
    for c in 3 6 8; do
      RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --config $c --tag c${c}_$lib >> $OUT/ab_s3q.txt 2>&1
    done
  done
done
tail -3 $OUT/par_t2.log
cat $OUT/ab_s3q.txt
