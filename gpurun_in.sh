timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_suite.log 2>&1; echo suite=$? >> gpurun_out/gpu_suite.log
timeout 600 python tools/decode_ab.py --cfg C4_128 --layers 4 prod s32 > gpurun_out/ab_c4_128.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C4_64 --layers 4 prod s32 > gpurun_out/ab_c4_64.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C5 prod s32 > gpurun_out/ab_c5.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C1 prod s32 > gpurun_out/ab_c1.log 2>&1
