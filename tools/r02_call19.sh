# round 2, call 19: C2 square/multiply A/B with the n0' slot: square FORM 5 / 3, chain unroll 4 / 16 (L = 6)
set -x
TAG=r02s
OUT=gpurun_out
mkdir -p $OUT
export AB_REPS=12
for r in 1 2 3; do
  python tools/ecm_ab.py time --L 6 --curves 4096 --B1 2000 base sq_f5 sq_f3 unr4 unr16 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
done
ls -la $OUT | tail -3
