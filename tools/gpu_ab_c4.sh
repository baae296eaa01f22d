#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_c4.txt
for round in 1 2; do for lib in exp_libs/*.so; do
  RKC_LIB=$lib timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag $(basename $lib .so) >> $OUT/ab_c4.txt 2>&1
done; done
RKC_LIB=exp_libs/c4_ahead4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -q -k "c4 or slot_stress or pool_sizes or 65536 or big" > $OUT/tests_ahead4.log 2>&1; echo "rc=$?" >> $OUT/tests_ahead4.log
cat $OUT/ab_c4.txt
