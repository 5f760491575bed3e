# round 2, call 20: L = 6 square unroll 16 in the product (mulmod GPU tests), chain-unroll A/B at L = 8 / 12 / 16
set -x
TAG=r02t
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_mulmod.py -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_mulmod.txt 2>&1
export AB_REPS=12
for r in 1 2; do
  python tools/ecm_ab.py time --L 6 --curves 4096 --B1 2000 base >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
  python tools/ecm_ab.py time --L 8 --curves 4096 --B1 2000 base l8_unr16 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
  python tools/ecm_ab.py time --L 12 --curves 4096 --B1 2000 base l12_unr4 l12_unr8 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
  python tools/ecm_ab.py time --L 16 --curves 4096 --B1 2000 base l16_unr4 >> $OUT/${TAG}_ab.jsonl 2>> $OUT/${TAG}_ab.err
done
ls -la $OUT | tail -3
