# round 2, call 5: parity of the square FORM 2 / mul_add tree (mulmod + ECM GPU tests), A/B of the square forms per width
set -x
mkdir -p gpurun_out
T=r02e
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt
timeout 1800 python -m pytest tests/test_gpu_mulmod.py tests/test_gpu_ecm.py -q -x -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.txt 2>&1
W=227328
python tools/ecm_ab.py time --L 6 --curves 1048576,$W base l6_f1 l6_f2 l6_f2m > gpurun_out/${T}_ab6.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 4 --curves 1048576,$W base l4_f1 l4_f2 > gpurun_out/${T}_ab4.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 8 --curves $W base l8_f1 l8_f2 > gpurun_out/${T}_ab8.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 12 --curves $W base l12_f1 l12_f2 > gpurun_out/${T}_ab12.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 16 --curves $W base l16_f1 l16_f2 > gpurun_out/${T}_ab16.jsonl 2>> gpurun_out/${T}_ab.err
ls -la gpurun_out | tail -12
