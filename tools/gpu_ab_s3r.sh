#!/bin/bash
# Session-3 A/B #18: big pools' density-based first probe (stats pass also takes the class-1 max);
# pacing margin floor 4096 and pacing lag 2.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3r.txt
RKC_LIB=exp_libs/u1_statsmax.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q -k "c4 or pool_sizes or 65536 or big or slot" > $OUT/par_u1.log 2>&1; echo "rc=$?" >> $OUT/par_u1.log
RKC_LIB=exp_libs/q6_lag2.so timeout 600 python -m pytest tests/test_gpu_pacing.py -q > $OUT/par_q6.log 2>&1; echo "rc=$?" >> $OUT/par_q6.log
for round in 1 2; do
  for lib in v0_head u1_statsmax; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3r.txt 2>&1
  done
  for lib in v0_head q5_floor4k q6_lag2; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3r.txt 2>&1
    for c in 3 6 8; do
      RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --config $c --tag c${c}_$lib >> $OUT/ab_s3r.txt 2>&1
    done
  done
done
tail -n 3 $OUT/par_u1.log $OUT/par_q6.log
cat $OUT/ab_s3r.txt
