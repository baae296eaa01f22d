#!/bin/bash
# Session-3 A/B #10: hot headers kept in L2 (evict_last loads in the light pass, evict_last
# stores in the step kernel's write-back).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3j.txt
RKC_LIB=exp_libs/k2_evs_hdr.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_k2.log 2>&1; echo "rc=$?" >> $OUT/par_k2.log
for round in 1 2; do
  for lib in n_head5 j1_hdr k1_evs k2_evs_hdr; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3j.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3j.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3j.txt
