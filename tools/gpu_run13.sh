#!/bin/bash
set -x
OUT=gpurun_out; mkdir -p $OUT
bash tools/gpu_ab_c4.sh > /dev/null 2>&1
RKC_LIB=exp_libs/c4_preload.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "c4 or slot_stress or pool_sizes" > $OUT/tests_preload.log 2>&1; echo "rc=$?" >> $OUT/tests_preload.log
timeout 2400 python tests/run_parity_1m.py --single-pool --config 4 --traces 10000 --steps 1024 --blocks 65536 --slots 16 16 128 --chunk 100 > $OUT/parity_c4_full.log 2>&1; echo "rc=$?" >> $OUT/parity_c4_full.log
ls -la $OUT
