#!/bin/bash
# Session-3 A/B #2: defaults (probe from registers, ranked light takes, crew L2 prefetch 4 ahead,
# big builds back to the out-of-line op paths) against variants.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3b.txt
for lib in n_head s_warpatom; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for lib in t_crew4 o_biginl; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c4 or pool_sizes or 65536 or big or slot" > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for round in 1 2; do
  for lib in a_base n_head s_warpatom; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3b.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3b.txt 2>&1
  done
  for lib in a_base n_head o_biginl p_pf2 q_pf3 r_pf4u4 t_crew4; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3b.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3b.txt
