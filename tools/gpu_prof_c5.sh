#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --set full --clock-control none --import-source on -k regex:"rkc_(step|light|step_overflow)_kernel" -s 384 -c 3 -o $OUT/prof_c5 python tools/profile_run.py --traces 1000000 > $OUT/prof_c5.log 2>&1
ls -la $OUT
