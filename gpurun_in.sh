timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "fused_search or assign" > gpurun_out/t18.log 2>&1; echo t18=$? > gpurun_out/rc17.txt
timeout 600 python tools/search_time.py C5 C3 C2 C4 > gpurun_out/search_time.log 2>&1
