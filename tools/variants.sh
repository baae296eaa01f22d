#!/bin/bash
# Build and bench several __launch_bounds__ occupancy variants of the step kernel on the GPU box.
# usage: bash tools/variants.sh 16 20 22
OUT=gpurun_out; mkdir -p $OUT
for occ in "$@"; do
  sed -i "s/__launch_bounds__(kWarpsPerCta \* 32, [0-9]*)/__launch_bounds__(kWarpsPerCta * 32, $occ)/" paper_2605_24259_b200/csrc/rkc_step_impl.cuh
  python paper_2605_24259_b200/build.py > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 1 > $OUT/variant_$occ.json 2> $OUT/variant_$occ.err
  python -c "import json; d=json.load(open('$OUT/variant_$occ.json')); print('occ $occ', '%.4e'%d['value'], 'launch_us %.1f'%d['roofline']['avg_launch_us'], 'frac %.3f'%d['roofline']['frac'])" >> $OUT/variants.txt 2>&1
done
cat $OUT/variants.txt
