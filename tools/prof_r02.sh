#!/bin/bash
# round-2 ncu evidence: --set full captures of the decode, quantize and window-score kernels
# (clock-control none), and the decode once more under --clock-control base
set -x
bash tools/prof_kernel.sh '^k_decode$' r02e 2
#bash tools/prof_kernel.sh k_quant r02q 2
#bash tools/prof_kernel.sh k_window_scores r02s 0
ARGS="--layers 2 --n-gen 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-ablation"
#ncu --set full --clock-control base --import-source on -k 'regex:^k_decode$' -s 2 -c 1 \
    -o gpurun_out/prof_r02db -f python bench.py $ARGS > gpurun_out/prof_ncu_r02db.log 2>&1
#ncu -i gpurun_out/prof_r02db.ncu-rep --page raw --csv > gpurun_out/prof_r02db.raw.csv 2>&1 || true
#ncu -i gpurun_out/prof_r02db.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_r02db.sass.csv 2>&1 || true
rm -f gpurun_out/*.ncu-rep
