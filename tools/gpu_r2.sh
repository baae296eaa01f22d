#!/bin/bash
# Round-2 GPU session: GPU tests, smoke, default bench (c5), a 2-rank bench on the one GPU.
set -x
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $OUT/smi.txt 2>&1
free -g > $OUT/free.txt 2>&1; lscpu > $OUT/lscpu.txt 2>&1; nproc >> $OUT/lscpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=20 > $OUT/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
if [ "${N2:-1}" = "1" ]; then
  RKC_BENCH_WATCHDOG=500 timeout 600 python bench.py --gpus 2 --steps 3 --no-cpu-baseline > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "bench n2 rc=$?" >> $OUT/bench_n2.err
fi
ls -la $OUT
