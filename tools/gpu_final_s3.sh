#!/bin/bash
# End-of-round GPU evidence for the committed build: ncu captures first (the bench's
# roofline.traffic is refreshed from them on the box), then GPU tests, smoke, the bench lines,
# the reference arm, the 10^6-trace single-pool parity run and a per-step profile.
set -x
OUT=gpurun_out; mkdir -p $OUT
python -c "from paper_2605_24259_b200 import build; build.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > $OUT/smi.txt 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light|step_overflow)_kernel" -s 384 -c 3 -o $OUT/prof_c5 python tools/profile_run.py --traces 1000000 > $OUT/prof_c5.log 2>&1
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light)_kernel" -s 200 -c 2 -o $OUT/prof_c4 python tools/profile_run.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 128 > $OUT/prof_c4.log 2>&1
python tools/ncu_traffic_json.py $OUT/prof_c5.ncu-rep profiles/ncu_step_kernel_c5.json "ncu --set full, steady-state c5 step (launches 384-386), round-2 final build" > $OUT/traffic_c5.log 2>&1
python tools/ncu_traffic_json.py $OUT/prof_c4.ncu-rep profiles/ncu_step_kernel_c4.json "ncu --set full, steady-state c4 step (launches 200-201), round-2 final build" > $OUT/traffic_c4.log 2>&1
cp profiles/ncu_step_kernel_c5.json profiles/ncu_step_kernel_c4.json $OUT/
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python tools/profile_run.py --traces 1000000 > $OUT/launches_c5.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $OUT/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $OUT/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for c in c5 c3 c4 c6 c8; do
  timeout 1500 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "rc=$?" >> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "rc=$?" >> $OUT/bench_reference.err
for r in 1 2; do timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 > $OUT/bench_n2_$r.json 2> $OUT/bench_n2_$r.err; echo "rc=$?" >> $OUT/bench_n2_$r.err; done
timeout 600 python tools/step_timing.py --traces 1000000 --reps 1 --per-step --tag c5_perstep > $OUT/perstep.txt 2>&1
timeout 600 python tools/step_timing.py --traces 1000000 --reps 1 --nop --per-step --tag c5_nop >> $OUT/perstep.txt 2>&1
timeout 2400 python tests/run_parity_1m.py --single-pool --chunk 50000 > $OUT/parity_1m_single_pool.log 2>&1; echo "rc=$?" >> $OUT/parity_1m_single_pool.log
ls -la $OUT
