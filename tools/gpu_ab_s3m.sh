#!/bin/bash
# Session-3 A/B #13: host-paced step grid (sized from the heavy count published 3 steps earlier).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3m.txt
RKC_LIB=exp_libs/p1_pacing.so timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/par_p1.log 2>&1; echo "rc=$?" >> $OUT/par_p1.log
for round in 1 2; do
  for lib in n_clean p1_pacing; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3m.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3m.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --config 6 --tag c6_$lib >> $OUT/ab_s3m.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --config 8 --tag c8_$lib >> $OUT/ab_s3m.txt 2>&1
  done
done
RKC_LIB=exp_libs/p1_pacing.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 1 --per-step --tag c5ps_pacing >> $OUT/ab_s3m.txt 2>&1
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3m.txt
