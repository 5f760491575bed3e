# round 2, call 18: ladder A/B at L = 4 (mul_add frame, canonical-input squares, loop unroll 2) and L = 6
# (canonical-input squares), C3-shaped inputs at B1 = 50000, whole waves (6 CTAs x 128 x 148 x 2)
set -x
TAG=r02r
OUT=gpurun_out
mkdir -p $OUT
export AB_MULMOD=0
for r in 1 2; do
  python tools/ecm_ab.py time --L 4 --curves 227328 --B1 50000 base l4_muladd l4_canon l4_unr2 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
  python tools/ecm_ab.py time --L 6 --curves 227328 --B1 50000 base l6_canon >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
done
ls -la $OUT | tail -4
