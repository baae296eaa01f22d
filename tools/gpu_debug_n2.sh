#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
python -c "from paper_2605_24259_b200 import build; build.build()"
timeout 600 python tools/debug_shard.py --first 500000 --n 500000 > $OUT/dbg_shard1.log 2>&1; echo "rc=$?" >> $OUT/dbg_shard1.log
timeout 600 python tools/debug_shard.py --first 0 --n 500000 > $OUT/dbg_shard0.log 2>&1; echo "rc=$?" >> $OUT/dbg_shard0.log
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "rc=$?" >> $OUT/bench_n2.err
timeout 900 python bench.py --gpus 2 --config c3 --steps 3 --warmup 3 > $OUT/bench_n2_c3.json 2> $OUT/bench_n2_c3.err; echo "rc=$?" >> $OUT/bench_n2_c3.err
tail -3 $OUT/dbg_shard*.log $OUT/bench_n2*.err
