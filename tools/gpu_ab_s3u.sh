#!/bin/bash
# Session-3 A/B #21: the mask apply's list built one iteration per taken key (dp4a rank bases).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3u.txt
RKC_LIB=exp_libs/z1_listbits.so timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/par_z1.log 2>&1; echo "rc=$?" >> $OUT/par_z1.log
for round in 1 2; do
  for lib in z0_head z1_listbits; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3u.txt 2>&1
    for c in 3 6 8; do
      RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --config $c --tag c${c}_$lib >> $OUT/ab_s3u.txt 2>&1
    done
  done
done
tail -3 $OUT/par_z1.log
cat $OUT/ab_s3u.txt
