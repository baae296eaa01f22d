#!/bin/bash
# Session-3 A/B #6 (big pools): interleaved 4-vector chunks per crew warp (per-chunk counts for
# the apply ranks), one 16-B read-back per vector in apply / touch.
OUT=gpurun_out; mkdir -p $OUT
: > $OUT/ab_s3f.txt
for lib in e1_ilv e2_ilv_vec d1_vec; do
  RKC_LIB=exp_libs/$lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefix_hits.py -x -q -k "c4 or pool_sizes or 65536 or big or slot" > $OUT/par_$lib.log 2>&1; echo "rc=$?" >> $OUT/par_$lib.log
done
for round in 1 2; do
  for lib in n_head2 d1_vec e1_ilv e2_ilv_vec; do
    RKC_LIB=exp_libs/$lib.so timeout 400 python tools/step_timing.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 256 --reps 2 --tag c4_$lib >> $OUT/ab_s3f.txt 2>&1
  done
done
tail -n 3 $OUT/par_*.log
cat $OUT/ab_s3f.txt
