#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for d in "$@"; do
  RKC_NVCC_EXTRA="-DRKC_DISPATCH=$d" python -c "import sys; sys.path.insert(0,'.'); from paper_2605_24259_b200 import build; build.build(force=True)" > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > $OUT/disp_$d.json 2> $OUT/disp_$d.err
  python -c "import json; d=json.load(open('$OUT/disp_$d.json')); print('dispatch $d', '%.4e'%d['value'], 'launch_us %.1f'%d['roofline']['avg_launch_us'], 'frac %.3f'%d['roofline']['frac'])" >> $OUT/dispatch.txt 2>&1
done
cat $OUT/dispatch.txt
