timeout 600 python tools/decode_ab.py --cfg C5 prod c2a c2b > gpurun_out/ab_c5.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C3 prod c2a c2b > gpurun_out/ab_c3.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C4 --layers 4 prod c2a c2b > gpurun_out/ab_c4.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C2 prod c2a c2b > gpurun_out/ab_c2.log 2>&1
WQ_VARIANT=c2a timeout 600 python tools/decode_err.py C1 C2 C3 C5 > gpurun_out/err_c2a.log 2>&1
