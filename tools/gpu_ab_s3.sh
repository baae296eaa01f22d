#!/bin/bash
# Session-3 A/B: mask-carrying probes (small pools), rank-parallel free-only takes (light pass,
# step kernel), crew L2 prefetch distance (big pools).  Parity subsets on the variants first,
# then step timing (µs per lockstep step, tools/step_timing.py).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3.txt
for lib in b_mask c_maskreg j_light10_free h_light; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
RKC_LIB=exp_libs/f_pf8.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c4 or pool_sizes or 65536 or big or slot" > $OUT/par_f_pf8.log 2>&1; echo "rc=$?" >> $OUT/par_f_pf8.log
for round in 1 2; do
  for lib in a_base b_mask c_maskreg d_mask_occ2 h_light i_light10 j_light10_free; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3.txt 2>&1
  done
  for lib in a_base e_pf4 f_pf8 g_pf16; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3.txt
