# round 2, call 2: GPU suite + smoke on the new tree, then ladder A/B round 2 (all widths)
set -x
mkdir -p gpurun_out
T=r02b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
python tools/ecm_ab.py time --L 4 --curves 1048576,131072 base l4_minb7 l4_minb8 l4_old > gpurun_out/${T}_ab4.jsonl 2>> gpurun_out/${T}_ab.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 6 --curves 1048576,131072 base l6_sqr1 l6_old l6_minb5 > gpurun_out/${T}_ab6.jsonl 2>> gpurun_out/${T}_ab.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 8 --curves 262144,131072 base l8_old l8_minb4 > gpurun_out/${T}_ab8.jsonl 2>> gpurun_out/${T}_ab.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 12 --curves 131072 base l12_old > gpurun_out/${T}_ab12.jsonl 2>> gpurun_out/${T}_ab.err
AB_MULMOD=0 python tools/ecm_ab.py time --L 16 --curves 131072 base l16_old > gpurun_out/${T}_ab16.jsonl 2>> gpurun_out/${T}_ab.err
ls -la gpurun_out | tail -20
