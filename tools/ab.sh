#!/bin/bash
# A/B timing of librkc variants in exp_libs/*.so (tools/step_timing.py), interleaved twice.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab.txt
for round in 1 2; do
  for lib in exp_libs/*.so; do
    RKC_LIB=$lib timeout 300 python tools/step_timing.py --tag $(basename $lib .so) $AB_ARGS >> $OUT/ab.txt 2>&1
  done
done
if [ -n "$AB_NOP" ]; then RKC_LIB=exp_libs/base.so timeout 300 python tools/step_timing.py --nop --tag nop_floor >> $OUT/ab.txt 2>&1; fi
cat $OUT/ab.txt
