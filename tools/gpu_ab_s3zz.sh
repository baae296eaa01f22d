#!/bin/bash
# Session-3 A/B #24: finish() bookkeeping in two 16-B loads; crew reclass bitmap in registers (c4).
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3zz.txt
RKC_LIB=exp_libs/zi_bucketcmp.so timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/par_zi.log 2>&1; echo "rc=$?" >> $OUT/par_zi.log
for round in 1 2; do
  for lib in zh_head zi_bucketcmp; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python tools/step_timing.py --traces 1000000 --reps 3 --tag c5_$lib >> $OUT/ab_s3zz.txt 2>&1
    for c in 3 6 8; do
      RKC_LIB=exp_libs/$lib.so timeout 300 python tools/step_timing.py --config $c --tag c${c}_$lib >> $OUT/ab_s3zz.txt 2>&1
    done
  done
  for lib in zh_head; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3zz.txt 2>&1
  done
done
tail -3 $OUT/par_zi.log
cat $OUT/ab_s3zz.txt
