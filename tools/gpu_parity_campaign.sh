#!/bin/bash
# Round-2 parity campaign in the bench's launch configuration (one pool per run):
# c6 and c8 at 10^6 traces, c7 slot stress at 100k traces, c4 at full length.
set -x
OUT=gpurun_out; mkdir -p $OUT
timeout 1800 python tests/run_parity_1m.py --single-pool --config 6 --chunk 50000 > $OUT/parity_1m_c6.log 2>&1; echo "rc=$?" >> $OUT/parity_1m_c6.log
timeout 1800 python tests/run_parity_1m.py --single-pool --config 8 --chunk 50000 > $OUT/parity_1m_c8.log 2>&1; echo "rc=$?" >> $OUT/parity_1m_c8.log
timeout 1200 python tests/run_parity_1m.py --single-pool --config 7 --traces 100000 --steps 400 --blocks 256 --slots 32 32 128 --chunk 20000 > $OUT/parity_100k_c7.log 2>&1; echo "rc=$?" >> $OUT/parity_100k_c7.log
timeout 1800 python tests/run_parity_1m.py --single-pool --config 4 --traces 320 --steps 1024 --blocks 65536 --slots 16 16 128 --u-range 12000 65536 --chunk 32 > $OUT/parity_c4_320.log 2>&1; echo "rc=$?" >> $OUT/parity_c4_320.log
timeout 900 python bench.py --config c8 > $OUT/bench_c8.json 2> $OUT/bench_c8.err; echo "rc=$?" >> $OUT/bench_c8.err
ls -la $OUT
