# round 2, call 6: GPU suite on the per-width FORM 2 product; A/B FORM 3 (no injection) per width; bench line
set -x
mkdir -p gpurun_out
T=r02f
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.txt 2>&1
W=227328
python tools/ecm_ab.py time --L 6 --curves 1048576,$W base l6_f3 > gpurun_out/${T}_ab6.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 4 --curves 1048576,$W base l4_f3 > gpurun_out/${T}_ab4.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 8 --curves $W base l8_f3 > gpurun_out/${T}_ab8.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 12 --curves $W base l12_f3 > gpurun_out/${T}_ab12.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 16 --curves $W base l16_f3 > gpurun_out/${T}_ab16.jsonl 2>> gpurun_out/${T}_ab.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${T}_bench.jsonl 2> gpurun_out/${T}_bench.err
ls -la gpurun_out | tail -12
