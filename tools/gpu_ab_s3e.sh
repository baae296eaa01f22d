#!/bin/bash
# Session-3 A/B #5 (big pools): tables preloaded for ADVANCE, crews of 16 warps, fp32 probe
# estimates, crew passes not unrolled.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3e.txt
RKC_LIB=exp_libs/c3_f32.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_c3_f32.log 2>&1; echo "rc=$?" >> $OUT/par_c3_f32.log
for lib in c1_preload c2_crew16 c4_u1 n_head; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c4 or pool_sizes or 65536 or big or slot" > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for round in 1 2; do
  for lib in n_head c3_f32; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3e.txt 2>&1
  done
  for lib in n_head c1_preload c2_crew16 c3_f32 c4_u1; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3e.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3e.txt
