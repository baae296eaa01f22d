#!/bin/bash
# e2e (host op stream) vs device-resident timing for each librkc variant in exp_libs/
for lib in exp_libs/*.so; do
  RKC_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 5 --e2e-steps 3 > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
  python -c "import json; d=json.load(open('gpurun_out/bench_e2e.json')); print('$(basename $lib .so)', 'value %.4e ms %.2f e2e %.4e ms %.2f' % (d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step']))"
done
