# round 2, call 26: C2 kernel occupancy with the n0' slot: 3 / 5 CTAs per SM (85 / 51 registers), 3 CTAs + unroll 16
set -x
TAG=r02z
OUT=gpurun_out
mkdir -p $OUT
export AB_REPS=12
for r in 1 2 3; do
  python tools/ecm_ab.py time --L 6 --curves 4096 --B1 2000 base mb3 mb5 mb3u16 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
done
