#!/bin/bash
# Session-3 A/B #19: light-pass free-only takes served from the lowest non-empty bitmap word
# without a scan when it holds the whole allocation.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3s.txt
RKC_LIB=exp_libs/w1_fafast.so timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/par_w1.log 2>&1; echo "rc=$?" >> $OUT/par_w1.log
for round in 1 2; do
  for lib in w0_head w1_fafast; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3s.txt 2>&1
    for c in 3 6 8; do
      RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --config $c --tag c${c}_$lib >> $OUT/ab_s3s.txt 2>&1
    done
  done
done
tail -3 $OUT/par_w1.log
cat $OUT/ab_s3s.txt
