#!/bin/bash
# Session-3 A/B #9 (light pass): two traces per thread, both traces' loads in flight together,
# one pair of CTA barriers for both.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3i.txt
for lib in i1_ilp2_8 i2_ilp2_6; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for round in 1 2; do
  for lib in n_head4 i1_ilp2_8 i2_ilp2_6; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3i.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3i.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3i.txt
RKC_LIB=exp_libs/n_head4.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 1 --per-step --tag c5_perstep >> $OUT/ab_s3i.txt 2>&1
RKC_LIB=exp_libs/n_head4.so timeout 600 python tools/step_timing.py --reps 1 --per-step --tag c3_perstep >> $OUT/ab_s3i.txt 2>&1
RKC_LIB=exp_libs/n_head4.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 1 --nop --per-step --tag c5_nop >> $OUT/ab_s3i.txt 2>&1
tail -3 $OUT/ab_s3i.txt
