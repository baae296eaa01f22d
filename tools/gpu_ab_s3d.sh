#!/bin/bash
# Session-3 A/B #4: ticket fields as uniform loads, counters as predicated shared reductions;
# then ncu captures of the current build (c4 crew step, c5 step).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3d.txt
for lib in a3_tku_red a1_tku; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for round in 1 2; do
  for lib in n_head a1_tku a2_red a3_tku_red; do
    RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --tag c3_$lib >> $OUT/ab_s3d.txt 2>&1
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3d.txt 2>&1
  done
done
bash tools/gpu_prof_s3.sh
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3d.txt
