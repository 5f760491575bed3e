# round 2, call 9: A/B of the square chain order 1 (FORM 4: high half added, FORM 5: injected) per width; sustained C3
set -x
mkdir -p gpurun_out
T=r02i
W=227328
python tools/ecm_ab.py time --L 4 --curves 1048576,$W base l4_f4 > gpurun_out/${T}_ab4.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 6 --curves 1048576,$W base l6_f4 l6_f5 > gpurun_out/${T}_ab6.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 8 --curves $W base l8_f4 l8_f5 > gpurun_out/${T}_ab8.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 12 --curves $W base l12_f4 l12_f5 > gpurun_out/${T}_ab12.jsonl 2>> gpurun_out/${T}_ab.err
python tools/ecm_ab.py time --L 16 --curves $W base l16_f4 l16_f5 > gpurun_out/${T}_ab16.jsonl 2>> gpurun_out/${T}_ab.err
python bench.py --gpus 1 --steps 5 --warmup 3 --no-sweep --no-cpu --ecm-curves 4194304 > gpurun_out/${T}_sustained_c3.jsonl 2> gpurun_out/${T}_sustained_c3.err
ls -la gpurun_out | tail -8
