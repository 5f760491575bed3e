# round 2, call 15: A/B of n0' parked in shared memory (MULMOD_N0_SMEM) in the C2 mulmod/square chains at
# L = 4/6/8 (alternating base/variant, 3 rounds), full ncu captures of the L = 12 and L = 16 ladders
set -x
TAG=r02o
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt
export AB_REPS=12
for r in 1 2 3; do
  for L in 6 4 8; do
    python tools/ecm_ab.py time --L $L --curves 16384 --B1 2000 base n0s$L >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
  done
done
cap() {  # name kernel-regex driver-args...
  local name=$1 re=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -c 1 -o /tmp/${TAG}_$name \
      python tools/prof_driver.py "$@" > $OUT/${TAG}_ncu_$name.log 2>&1
  ncu -i /tmp/${TAG}_$name.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_${name}_raw.csv 2>/dev/null
  rm -f /tmp/${TAG}_$name.ncu-rep
}
cap ecm_l16 ecm_stage1_kernel ecm --L 16 --curves 75776 --B1 2000 --reps 1
cap ecm_l12 ecm_stage1_kernel ecm --L 12 --curves 113664 --B1 2000 --reps 1
ls -la $OUT | tail -8
