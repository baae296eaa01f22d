#!/bin/bash
# compute-sanitizer on the final build: memcheck over the f3 + paper parity subsets,
# racecheck and synccheck over smoke() (small shapes: the tools slow kernels 10-100x).
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_prefix_hits.py tests/test_gpu_parity.py -x -q -k "hit_litmus or o128 or injection or paper_litmus or pool_sizes or slot_limits or c4_subset" > $OUT/sanitize_memcheck.log 2>&1; echo "rc=$?" >> $OUT/sanitize_memcheck.log
timeout 900 $CS --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitize_racecheck.log 2>&1; echo "rc=$?" >> $OUT/sanitize_racecheck.log
timeout 900 $CS --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitize_synccheck.log 2>&1; echo "rc=$?" >> $OUT/sanitize_synccheck.log
