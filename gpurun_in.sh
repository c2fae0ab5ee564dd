timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/t_h.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C5 --rounds 8 prod h0 > gpurun_out/ab_c5.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C3 prod h0 > gpurun_out/ab_c3.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C2 prod h0 > gpurun_out/ab_c2.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C4 --layers 4 prod h0 > gpurun_out/ab_c4.log 2>&1
