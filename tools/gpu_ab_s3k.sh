#!/bin/bash
# Session-3 A/B #11: the step's heavy items spread evenly over the grid (empty CTAs between the
# busy ones instead of a dispatch-bound tail).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3k.txt
RKC_LIB=exp_libs/l1_spread.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_l1.log 2>&1; echo "rc=$?" >> $OUT/par_l1.log
RKC_LIB=exp_libs/m1_tmask.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q -k "c4 or pool_sizes or 65536 or big or slot" > $OUT/par_m1.log 2>&1; echo "rc=$?" >> $OUT/par_m1.log
for round in 1 2; do
  for lib in n_head6 m1_tmask; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3k.txt 2>&1
  done
  for lib in n_head6 l1_spread; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3k.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3k.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --config 6 --tag c6_$lib >> $OUT/ab_s3k.txt 2>&1
  done
done
for lib in n_head6 l1_spread; do
  RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 1 --per-step --tag c5ps_$lib >> $OUT/ab_s3k.txt 2>&1
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3k.txt
