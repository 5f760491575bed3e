# round 2, call 21: final tree (n0' slot, L = 6 square unroll 16, best-of-2 ECM widths): GPU suite + smoke,
# the driver's default bench command (twice), reference arm, ncu launch list, compute-sanitizer of every launch
# path, sustained C2 (1600 steps, clocks sampled)
set -x
TAG=r02u
OUT=gpurun_out
mkdir -p $OUT/${TAG}_sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
python bench.py > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
python bench.py > $OUT/${TAG}_bench_b.jsonl 2> $OUT/${TAG}_bench_b.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_bench_reference.jsonl 2> $OUT/${TAG}_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --no-cpu --no-sweep --steps 3 --warmup 3 > $OUT/${TAG}_launches_bench.jsonl 2>&1
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_driver.py > $OUT/${TAG}_sanitizer/$tool.txt 2>&1
done
python bench.py --steps 1600 --warmup 5 --no-ecm --no-sweep --no-cpu > $OUT/${TAG}_sustained_c2.jsonl 2> $OUT/${TAG}_sustained_c2.err
ls -la $OUT | tail -14; for f in $OUT/${TAG}_sanitizer/*.txt; do tail -n 2 $f; done
