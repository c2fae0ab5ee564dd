timeout 600 python tools/decode_ab.py --cfg C5 --rounds 8 prod rr1 rr5 > gpurun_out/ab_c5.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C3 prod rr1 rr5 > gpurun_out/ab_c3.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C4 --layers 4 prod rr1 rr5 > gpurun_out/ab_c4.log 2>&1
