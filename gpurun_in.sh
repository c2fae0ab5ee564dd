timeout 600 python tools/decode_ab.py --layers 8 --tokens 10 --rounds 5 prod cr80 lov1k lov2k lov3k lov2o > gpurun_out/ab7.log 2>&1
timeout 300 python tools/decode_ab.py --cfg C2 --layers 12 --tokens 10 --rounds 5 prod cr80 lov1k lov2k lov3k lov2o > gpurun_out/ab7_c2.log 2>&1
timeout 300 python tools/decode_ab.py --cfg C3 --layers 8 --tokens 6 --rounds 4 prod cr80 lov1k lov2k lov3k lov2o > gpurun_out/ab7_c3.log 2>&1
