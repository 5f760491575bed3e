# round 2, call 12: host-buffer chunk ramp (abi.cu pipeline_chunks): host-buffer parity tests, bench (e2e), multi-rank bench on one GPU
set -x
TAG=r02m
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_mulmod.py -q -p no:cacheprovider -k "host_buffers or c2_full or max_size" > $OUT/${TAG}_pytest_host.txt 2>&1
python bench.py --gpus 1 --steps 20 --warmup 5 > $OUT/${TAG}_bench.jsonl 2> $OUT/${TAG}_bench.err
python bench.py --gpus 1 --steps 20 --warmup 5 --no-ecm --no-sweep --no-cpu > $OUT/${TAG}_bench_b.jsonl 2> $OUT/${TAG}_bench_b.err
ECM_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29561 \
   bench.py --gpus 8 --steps 3 --warmup 3 --count 1048576 --ecm-curves 131072 --no-sweep > $OUT/${TAG}_torchrun8_gloo_onegpu.jsonl 2> $OUT/${TAG}_torchrun8.err
ls -la $OUT | tail -6
