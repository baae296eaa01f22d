#!/bin/bash
# Session-3 A/B #28: pacing margin 1/128 and 1/256 of the traces.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s4a.txt
RKC_LIB=exp_libs/zk_shift7.so timeout 600 python -m pytest tests/test_gpu_pacing.py -q > $OUT/par_zk.log 2>&1; echo "rc=$?" >> $OUT/par_zk.log
for round in 1 2; do
  for lib in zj_head zk_shift7 zl_shift8; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s4a.txt 2>&1
    for c in 3 8; do
      RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --config $c --tag c${c}_$lib >> $OUT/ab_s4a.txt 2>&1
    done
  done
done
tail -3 $OUT/par_zk.log
cat $OUT/ab_s4a.txt
