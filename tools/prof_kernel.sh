#!/bin/bash
# ncu capture of one launch of kernel <regex> inside a short bench run (1 GPU).
# usage: tools/prof_kernel.sh <regex> <tag> <skip> [extra bench args]
set -e
RE=$1; TAG=$2; SKIP=${3:-2}; shift 3 || true
mkdir -p gpurun_out
ARGS="--layers 2 --n-gen 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-ablation $*"
python bench.py $ARGS > gpurun_out/prof_plain_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$RE -s $SKIP -c 1 \
    -o gpurun_out/prof_$TAG -f python bench.py $ARGS > gpurun_out/prof_ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_$TAG.ncu-rep --page details --csv > gpurun_out/prof_$TAG.details.csv 2>&1 || true
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_$TAG.raw.csv 2>&1 || true
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$TAG.sass.csv 2>&1 || true
