# round 2, call 11: A/B of x0/a24 in shared memory with the swap-free step (frees 2L registers) x square form x occupancy
set -x
mkdir -p gpurun_out
T=r02k
W=227328
AB_MULMOD=0 python tools/ecm_ab.py time --L 6 --curves 1048576,$W base l6_f4s l6_f3s l6_f4s7 > gpurun_out/${T}_ab6.jsonl 2>> gpurun_out/${T}_ab.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 4 --curves 1048576,$W base l4_f4s l4_f4s8 > gpurun_out/${T}_ab4.jsonl 2>> gpurun_out/${T}_ab.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 8 --curves 1048576,$W base l8_f4s l8_f4s5 > gpurun_out/${T}_ab8.jsonl 2>> gpurun_out/${T}_ab.err
ls -la gpurun_out | tail -4
