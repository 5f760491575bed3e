# round 2, call 7: final-form product: GPU suite + smoke, lazy-bound debug build, bench line, ncu launch list
# of the default bench command, full ncu captures (C2 mulmod, square mode, C3-shaped ladders at L = 4/6/8)
set -x
TAG=r02g
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $OUT/${TAG}_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
timeout 1200 python tools/debug_bounds.py > $OUT/${TAG}_debug_bounds.json 2> $OUT/${TAG}_debug_bounds.err
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --no-cpu --no-sweep --steps 5 --warmup 3 > $OUT/${TAG}_launches_bench.jsonl 2>&1
cap() {  # name kernel-regex driver-args...
  local name=$1 re=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -c 1 -o /tmp/${TAG}_$name \
      python tools/prof_driver.py "$@" > $OUT/${TAG}_ncu_$name.log 2>&1
  ncu -i /tmp/${TAG}_$name.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_${name}_raw.csv 2>/dev/null
  rm -f /tmp/${TAG}_$name.ncu-rep
}
cap mulmod mulmod_batch_kernel mulmod --sliced --reps 1
cap sqr mulmod_batch_kernel mulmod --sliced --flags 2 --reps 1
cap ecm_l6 ecm_stage1_kernel ecm --curves 227328 --B1 2000 --reps 1
cap ecm_l4 ecm_stage1_kernel ecm --L 4 --curves 227328 --B1 2000 --reps 1
cap ecm_l8 ecm_stage1_kernel ecm --L 8 --curves 227328 --B1 2000 --reps 1
ls -la $OUT | tail -30
