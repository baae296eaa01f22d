#!/bin/bash
# ncu --set full of one steady-state c4 step (crew kernel) and one c5 step, current build.
OUT=gpurun_out; mkdir -p $OUT
python -c "from paper_2605_24259_b200 import build; build.build()"
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light)_kernel" -s 200 -c 2 -o $OUT/prof_c4_s3 python tools/profile_run.py --config 4 --traces 10000 --blocks 65536 --objects 128 --steps 128 > $OUT/prof_c4_s3.log 2>&1
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light|step_overflow)_kernel" -s 384 -c 3 -o $OUT/prof_c5_s3 python tools/profile_run.py --traces 1000000 > $OUT/prof_c5_s3.log 2>&1
ls -la $OUT
