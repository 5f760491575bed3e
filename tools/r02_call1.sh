set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_gpu.txt
python tools/ecm_ab.py time --curves 1048576,131072 base sel sqr2 selsqr2 nocap nocapsel nocapsqr2 > gpurun_out/r02a_ab6.jsonl 2> gpurun_out/r02a_ab6.err
python tools/ecm_ab.py time --L 4 --curves 1048576,131072 base sel4 sqr2_4 selsqr2_4 > gpurun_out/r02a_ab4.jsonl 2> gpurun_out/r02a_ab4.err
for L in 4 16; do
ncu --set full --clock-control none --import-source on -k regex:ecm_stage1_kernel -c 1 -o /tmp/r02a_ecm_l$L python tools/prof_driver.py ecm --L $L --curves 131072 --B1 2000 --reps 1 > gpurun_out/r02a_ncu_ecm_l$L.log 2>&1
ncu -i /tmp/r02a_ecm_l$L.ncu-rep --page raw --csv > gpurun_out/r02a_ncu_ecm_l${L}_raw.csv 2>/dev/null
ncu -i /tmp/r02a_ecm_l$L.ncu-rep --page source --csv > gpurun_out/r02a_ncu_ecm_l${L}_source.csv 2>/dev/null
done
ls -la gpurun_out
