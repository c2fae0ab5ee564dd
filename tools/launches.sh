#!/bin/bash
# ncu launch list (per-launch device time, cold-cache, serialised) of a short bench run
set -e
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu --no-ablation --n-gen 2"
python bench.py $ARGS > gpurun_out/launch_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/launch_ncu.log 2>&1
