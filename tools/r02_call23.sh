# round 2, call 23: the Table 5 analogue (tools/ablation.py) re-run on the final tree
set -x
TAG=r02w
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python tools/ablation.py > $OUT/${TAG}_ablation.json 2> $OUT/${TAG}_ablation.err
head -c 3000 $OUT/${TAG}_ablation.json
