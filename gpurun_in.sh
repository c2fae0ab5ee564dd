timeout 1200 bash tools/run_cfgs.sh > gpurun_out/run_cfgs.log 2>&1
bash tools/prof_kernel.sh '^k_decode$' r02f 2
rm -f gpurun_out/*.ncu-rep
