set -x
OUT=gpurun_out
mkdir -p $OUT
python -c "from paper_2605_24259_b200 import build; build.build()"
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"rkc_(step|light)_kernel" -s 256 -c 2 -o $OUT/prof_step1 python tools/profile_run.py > $OUT/prof1.log 2>&1; echo "rc=$?" >> $OUT/prof1.log
ls -la $OUT/prof_step1*
