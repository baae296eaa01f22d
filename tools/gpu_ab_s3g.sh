#!/bin/bash
# Session-3 A/B #7 (light pass): bucket counters one 128-B line apart (less same-sector atomic
# contention), + per-warp atomics, light pass at 40 registers (12 CTAs per SM).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3g.txt
for lib in f1_spread f2_spread_wa f3_light12; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for round in 1 2; do
  for lib in n_head3 f1_spread f2_spread_wa f3_light12; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3g.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3g.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3g.txt
