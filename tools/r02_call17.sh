# round 2, call 17: final tree (n0' slot per width, device-staged ECM seeds + deferred decode): GPU suite +
# smoke, the driver's default bench command, reference arm, ncu launch list, 8-rank gloo-on-one-GPU bench
set -x
TAG=r02q
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/${TAG}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1
python bench.py > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/${TAG}_bench_b.jsonl 2> $OUT/${TAG}_bench_b.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_bench_reference.jsonl 2> $OUT/${TAG}_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --no-cpu --no-sweep --steps 3 --warmup 3 > $OUT/${TAG}_launches_bench.jsonl 2>&1
ECM_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29561 \
   bench.py --gpus 8 --steps 3 --warmup 3 --count 1048576 --ecm-curves 131072 --no-sweep > $OUT/${TAG}_torchrun8_gloo_onegpu.jsonl 2> $OUT/${TAG}_torchrun8.err
ls -la $OUT | tail -12
