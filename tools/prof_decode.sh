#!/bin/bash
# ncu capture of one wq_decode_attention launch inside a short bench run (1 GPU).
# usage: tools/prof_decode.sh <tag> [extra bench args]
set -e
TAG=${1:-r01}; shift || true
mkdir -p gpurun_out
ARGS="--layers 2 --n-gen 1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-ablation $*"
python bench.py $ARGS > gpurun_out/prof_plain_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode -s 2 -c 1 \
    -o gpurun_out/prof_decode_$TAG -f python bench.py $ARGS > gpurun_out/prof_ncu_$TAG.log 2>&1
ncu -i gpurun_out/prof_decode_$TAG.ncu-rep --page details --csv > gpurun_out/prof_decode_$TAG.details.csv 2>&1 || true
ncu -i gpurun_out/prof_decode_$TAG.ncu-rep --page raw --csv > gpurun_out/prof_decode_$TAG.raw.csv 2>&1 || true
