#!/bin/bash
# Session-3 A/B #3: c4 regression bisect (round-2 commits, no crew prefetch), and small-pool
# variants: reverse ticket order, two items per one-warp CTA (second ticket loaded ahead).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3c.txt
for lib in u_rev v_items2 n_head; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for round in 1 2; do
  for lib in n_head u_rev v_items2; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3c.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3c.txt 2>&1
  done
  for lib in w_9d6c x_c289 y_abdd z_6fce m_nopf n_head; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3c.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3c.txt
