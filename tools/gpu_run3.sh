set -x
OUT=gpurun_out; mkdir -p $OUT
bash tools/gpu_ab.sh > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > $OUT/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $OUT/gpu_tests.log
RKC_BENCH_WATCHDOG=400 timeout 600 python bench.py --gpus 2 --steps 3 --config c3 --no-cpu-baseline > $OUT/bench_n2.json 2> $OUT/bench_n2.err; echo "bench n2 rc=$?" >> $OUT/bench_n2.err
ls -la $OUT
