# round 2, call 27: L = 4 (C4's 128-bit width) chain A/B: unroll 16 / 4, 5 / 6 CTAs per SM
set -x
TAG=r02aa
OUT=gpurun_out
mkdir -p $OUT
export AB_REPS=12
for r in 1 2 3; do
  python tools/ecm_ab.py time --L 4 --curves 4096 --B1 2000 base l4_u16 l4_u4 l4_mb5 l4_mb6 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
done
