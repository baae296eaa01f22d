#!/bin/bash
# Session-3 A/B #22 (big pools): crew prefetch batched (one instruction per 8 vectors, one line per lane).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3v.txt
RKC_LIB=exp_libs/z2_pfbatch.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q -k "c4 or pool_sizes or 65536 or big or slot" > $OUT/par_z2.log 2>&1; echo "rc=$?" >> $OUT/par_z2.log
for round in 1 2; do
  for lib in z0b_head z2_pfbatch z3_pfbatch0; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3v.txt 2>&1
  done
done
tail -3 $OUT/par_z2.log
cat $OUT/ab_s3v.txt
