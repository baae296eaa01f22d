#!/bin/bash
# Round-2 evidence on the committed build: GPU tests, smoke, benches (c5 default, c3, c6, c4),
# the 10^6-trace single-pool parity run, compute-sanitizer on small shapes.
set -x
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $OUT/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > $OUT/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "rc=$?" >> $OUT/bench_c5.err
timeout 900 python bench.py --config c3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err; echo "rc=$?" >> $OUT/bench_c3.err
timeout 900 python bench.py --config c6 > $OUT/bench_c6.json 2> $OUT/bench_c6.err; echo "rc=$?" >> $OUT/bench_c6.err
timeout 1500 python bench.py --config c4 > $OUT/bench_c4.json 2> $OUT/bench_c4.err; echo "rc=$?" >> $OUT/bench_c4.err
timeout 900 python bench.py --config c8 > $OUT/bench_c8.json 2> $OUT/bench_c8.err; echo "rc=$?" >> $OUT/bench_c8.err
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "rc=$?" >> $OUT/bench_reference.err
timeout 2400 python tests/run_parity_1m.py --single-pool --chunk 50000 > $OUT/parity_1m_single_pool.log 2>&1; echo "rc=$?" >> $OUT/parity_1m_single_pool.log
# compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset)
ls -la $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light|step_overflow)_kernel" -s 384 -c 3 -o $OUT/prof_c5 python tools/profile_run.py --traces 1000000 > $OUT/prof_c5.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python tools/profile_run.py --traces 1000000 > $OUT/launches_c5.log 2>&1
