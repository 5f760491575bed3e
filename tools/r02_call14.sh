# round 2, call 14: final tree: GPU suite + smoke, the driver's default bench command, ncu launch list of it
set -x
TAG=r02n
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
python bench.py > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_bench_reference.jsonl 2> $OUT/${TAG}_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --no-cpu --no-sweep --steps 3 --warmup 3 > $OUT/${TAG}_launches_bench.jsonl 2>&1
ls -la $OUT | tail -8
