# round 2, call 3: GPU suite + smoke, default bench line, 8-rank gloo-on-one-GPU bench, ladder A/B (L 8/12/16)
set -x
mkdir -p gpurun_out
T=r02c
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.jsonl 2> gpurun_out/${T}_bench.err
ECM_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29561 \
   bench.py --gpus 8 --steps 3 --warmup 3 --count 1048576 --ecm-curves 131072 --no-sweep > gpurun_out/${T}_torchrun8_gloo_onegpu.jsonl 2> gpurun_out/${T}_torchrun8.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 8 --curves 262144 base l8_smem4 l8_sqr0 > gpurun_out/${T}_ab8.jsonl 2>> gpurun_out/${T}_ab.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 12 --curves 131072 base l12_sel l12_sqr1 l12_smem4 > gpurun_out/${T}_ab12.jsonl 2>> gpurun_out/${T}_ab.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 16 --curves 131072 base l16_sel l16_sqr1 l16_smem3 > gpurun_out/${T}_ab16.jsonl 2>> gpurun_out/${T}_ab.err
ls -la gpurun_out | tail -12
