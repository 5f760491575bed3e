# round 2, call 10: final per-width square forms: GPU suite + smoke, lazy-bound debug build, bench line, ncu square capture
set -x
TAG=r02j
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
timeout 1200 python tools/debug_bounds.py > $OUT/${TAG}_debug_bounds.json 2> $OUT/${TAG}_debug_bounds.err
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mulmod_batch_kernel -c 1 -o /tmp/${TAG}_sqr \
    python tools/prof_driver.py mulmod --sliced --flags 2 --reps 1 > $OUT/${TAG}_ncu_sqr.log 2>&1
ncu -i /tmp/${TAG}_sqr.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_sqr_raw.csv 2>/dev/null
ls -la $OUT | tail -8
