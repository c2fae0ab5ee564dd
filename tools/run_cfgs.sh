set -x
python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
for c in C1 C2 C3 C4; do python bench.py --config $c --no-cpu --no-e2e --no-ablation > gpurun_out/r02_bench_$c.json 2>> gpurun_out/r02_cfgs.err; done
bash tools/launches.sh
