# round 2, call 8: compute-sanitizer on the final build, C5 whole on one GPU, sustained C3 (4M curves, clocks sampled)
set -x
T=r02h
OUT=gpurun_out
mkdir -p $OUT/${T}_sanitizer
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_driver.py > $OUT/${T}_sanitizer/$tool.txt 2>&1
done
timeout 900 python tools/c5_full.py --out $OUT/${T}_c5_full.json > $OUT/${T}_c5_full.log 2>&1
python bench.py --gpus 1 --steps 5 --warmup 3 --no-sweep --no-cpu --ecm-curves 4194304 > $OUT/${T}_sustained_c3.jsonl 2> $OUT/${T}_sustained_c3.err
ls -la $OUT | tail; for f in $OUT/${T}_sanitizer/*.txt; do tail -n 2 $f; done
