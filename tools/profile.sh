#!/bin/bash
# Run on the GPU box (gpurun): bench line, launch list of the bench command, full ncu captures
# of the two hot kernels.  Outputs land in gpurun_out/ (copied to profiles/ by hand).
set -x
TAG=${TAG:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $OUT/${TAG}_gpu.txt
python bench.py ${BENCH_ARGS} > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
tail -3 $OUT/${TAG}_bench.err
if [ -z "$NO_NCU" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --ecm-curves 131072 > $OUT/${TAG}_launches_bench.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k regex:mulmod_batch_kernel -c 1 \
    -o $OUT/${TAG}_mulmod python tools/prof_driver.py mulmod --reps 1 > $OUT/${TAG}_ncu_mulmod.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ecm_stage1_kernel -c 1 \
    -o $OUT/${TAG}_ecm python tools/prof_driver.py ecm --curves 32768 --reps 1 > $OUT/${TAG}_ncu_ecm.log 2>&1
fi
ls -la $OUT
