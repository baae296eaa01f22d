#!/bin/bash
# Session-3 A/B #12: items spread over the grid only while pools fill (H < 3/4 G); overflow grid
# of 592 CTAs.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3l.txt
RKC_LIB=exp_libs/o4_ctrlanes.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_o4.log 2>&1; echo "rc=$?" >> $OUT/par_o4.log
RKC_LIB=exp_libs/o3_both.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_o3.log 2>&1; echo "rc=$?" >> $OUT/par_o3.log
for round in 1 2; do
  for lib in n_clean o1_spreadfill o2_ovf592 o3_both o4_ctrlanes; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3l.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3l.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3l.txt
