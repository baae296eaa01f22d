#!/bin/bash
# ncu evidence for round 2: launch lists + one --set full capture of a steady-state
# lockstep step (light + step + overflow) for c5 and c4.
set -x
OUT=gpurun_out; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c5.csv python tools/profile_run.py --traces 1000000 > $OUT/launches_c5.log 2>&1
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light|step_overflow)_kernel" -s 384 -c 3 -o $OUT/prof_c5 python tools/profile_run.py --traces 1000000 > $OUT/prof_c5.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches_c4.csv python tools/profile_run.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 128 > $OUT/launches_c4.log 2>&1
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light)_kernel" -s 200 -c 2 -o $OUT/prof_c4 python tools/profile_run.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 128 > $OUT/prof_c4.log 2>&1
ls -la $OUT
