# round 2, call 24: full ncu capture of the final C2 square kernel (n0' slot, unroll 16)
set -x
TAG=r02x
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mulmod_batch_kernel -c 1 -o /tmp/${TAG}_sqr \
    python tools/prof_driver.py mulmod --sliced --flags 2 --reps 1 > $OUT/${TAG}_ncu_sqr.log 2>&1
ncu -i /tmp/${TAG}_sqr.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_sqr_raw.csv 2>/dev/null
ls -la $OUT | tail -3
