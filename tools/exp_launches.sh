for lib in base new exact; do
RKC_LIB=exp_libs/$lib.so timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/l_$lib.csv python tools/step_timing.py --reps 0 > /dev/null 2>&1
done
