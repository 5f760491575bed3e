# round 2, call 25: GPU suite + smoke + default bench on the committed final tree
set -x
TAG=r02y
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
python bench.py > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
tail -n 1 $OUT/${TAG}_pytest_gpu.txt; tail -n 1 $OUT/${TAG}_smoke.txt
