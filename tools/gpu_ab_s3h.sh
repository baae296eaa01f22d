#!/bin/bash
# Session-3 A/B #8: tickets (and the request records of heavy traces) kept in L2 with an
# evict_last policy written / prefetched by the light pass.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3h.txt
for lib in g2_evl_rq; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for round in 1 2; do
  for lib in n_head4 g1_evl g2_evl_rq; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3h.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3h.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3h.txt
: > $OUT/ab_s3h_c4.txt
for round in 1 2; do
  for lib in n_head4 h1_pf6 h2_pf3; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3h_c4.txt 2>&1
  done
done
cat $OUT/ab_s3h_c4.txt
