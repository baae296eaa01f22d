#!/bin/bash
# Session-3 A/B #20: victims' meta lines prefetched (L1 + ld.ca / L2) right after the exact probe.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3t.txt
RKC_LIB=exp_libs/y1_metapf.so timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/par_y1.log 2>&1; echo "rc=$?" >> $OUT/par_y1.log
for round in 1 2; do
  for lib in y0_head y1_metapf y2_metapf_l2; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3t.txt 2>&1
    for c in 3 6; do
      RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --config $c --tag c${c}_$lib >> $OUT/ab_s3t.txt 2>&1
    done
  done
done
tail -3 $OUT/par_y1.log
cat $OUT/ab_s3t.txt
