# round 2, call 4 (re-entry): GPU suite + smoke on HEAD, ncu source captures of C1 / C3 for the setup/tail share
set -x
mkdir -p gpurun_out
T=r02d
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
for C in C1 C3; do
  if [ $C = C1 ]; then ARGS="--cfg C1 --curves 256 --B1 2000"; else ARGS="--cfg C3 --curves 16384 --B1 50000"; fi
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ecm_stage1 -c 1 -o /tmp/${T}_ncu_$C python tools/prof_driver.py ecm $ARGS --reps 1 > gpurun_out/${T}_ncu_$C.log 2>&1
  ncu -i /tmp/${T}_ncu_$C.ncu-rep --page raw --csv > gpurun_out/${T}_ncu_ecm_${C}_raw.csv 2>/dev/null
  ncu -i /tmp/${T}_ncu_$C.ncu-rep --page source --csv > gpurun_out/${T}_ncu_ecm_${C}_source.csv 2>/dev/null
  python tools/ncu_regions.py gpurun_out/${T}_ncu_ecm_${C}_source.csv --json > gpurun_out/${T}_regions_$C.json 2>&1
done
ls -la gpurun_out | tail -20
