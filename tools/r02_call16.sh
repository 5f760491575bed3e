# round 2, call 16: n0' shared-memory slot as the L = 6 default (and L = 4 square): GPU suite + smoke,
# A/B against the register form (sliced + AoS), the slot at L = 12/16, bench line, ncu of the C2 kernels
set -x
TAG=r02p
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
export AB_REPS=12
for r in 1 2; do
  AB_AOS=1 python tools/ecm_ab.py time --L 6 --curves 4096 --B1 2000 base n0off6 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
  python tools/ecm_ab.py time --L 12 --curves 4096 --B1 2000 base n0s12 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
  python tools/ecm_ab.py time --L 16 --curves 4096 --B1 2000 base n0s16 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
done
python bench.py > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
cap() {  # name kernel-regex driver-args...
  local name=$1 re=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -c 1 -o /tmp/${TAG}_$name \
      python tools/prof_driver.py "$@" > $OUT/${TAG}_ncu_$name.log 2>&1
  ncu -i /tmp/${TAG}_$name.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_${name}_raw.csv 2>/dev/null
  rm -f /tmp/${TAG}_$name.ncu-rep
}
cap mulmod mulmod_batch_kernel mulmod --sliced --reps 1
cap sqr mulmod_batch_kernel mulmod --sliced --flags 2 --reps 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --no-cpu --no-sweep --steps 3 --warmup 3 > $OUT/${TAG}_launches_bench.jsonl 2>&1
ls -la $OUT | tail -12
