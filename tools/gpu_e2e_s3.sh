#!/bin/bash
# e2e stability of the host-op-stream replay with and without grid pacing (3 bench runs each).
OUT=gpurun_out; mkdir -p $OUT
for r in 1 2 3; do
  for lib in x0_head x1_nohostpace; do
    RKC_LIB=exp_libs/$lib.so timeout 600 python bench.py --no-cpu-baseline > $OUT/e2e_c5_${lib}_$r.json 2> $OUT/e2e_c5_${lib}_$r.err
    RKC_LIB=exp_libs/$lib.so timeout 600 python bench.py --config c3 --no-cpu-baseline > $OUT/e2e_c3_${lib}_$r.json 2> $OUT/e2e_c3_${lib}_$r.err
  done
done
for f in $OUT/e2e_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); e=d['e2e']; print('$f', round(d['ms_per_step'],1), [round(x,1) for x in e['passes_ms']], '%.3e'%e['value'])"; done
