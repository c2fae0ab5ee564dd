timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_suite.log 2>&1; echo suite=$? >> gpurun_out/gpu_suite.log
timeout 1200 bash tools/run_cfgs.sh > gpurun_out/run_cfgs.log 2>&1
