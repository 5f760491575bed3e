#!/bin/bash
# Run on the GPU box (gpurun): bench line, ncu launch list of the exact default bench command,
# full ncu captures of the hot kernels exported to CSV (raw metrics + per-instruction source
# view).  The .ncu-rep files are deleted on the box (gpurun returns <= 64 MiB).
set -x
TAG=${TAG:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $OUT/${TAG}_gpu.txt
python bench.py > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
if [ -z "$NO_NCU" ]; then
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --no-cpu > $OUT/${TAG}_launches_bench.jsonl 2>&1
cap() {  # name kernel-regex driver-args...
  local name=$1 re=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$re -c 1 -o /tmp/${TAG}_$name \
      python tools/prof_driver.py "$@" > $OUT/${TAG}_ncu_$name.log 2>&1
  ncu -i /tmp/${TAG}_$name.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$name.ncu-rep --page source --csv > $OUT/${TAG}_ncu_${name}_source.csv 2>/dev/null
  rm -f /tmp/${TAG}_$name.ncu-rep
}
cap mulmod mulmod_batch_kernel mulmod --sliced --reps 1
cap mulmod_aos mulmod_batch_kernel mulmod --reps 1
cap sqr mulmod_batch_kernel mulmod --sliced --flags 2 --reps 1
cap k1 mulmod_ mulmod --iters 1 --reps 1
cap k1_sliced mulmod_ mulmod --sliced --iters 1 --reps 1
cap ecm ecm_stage1_kernel ecm --curves 1048576 --B1 2000 --reps 1
cap ecm_c1 ecm_stage1_coop ecm --cfg C1 --curves 256 --B1 2000 --reps 1
cap ecm_small ecm_stage1_kernel ecm --curves 1048576 --B1 2000 --flags 32768 --reps 1
cap mulmod_l16 mulmod_batch_kernel mulmod --sliced --L 16 --count 4194304 --reps 1
fi
ls -la $OUT
