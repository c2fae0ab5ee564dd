timeout 600 python tools/decode_ab.py --layers 8 --tokens 10 --rounds 5 prod s40 > gpurun_out/ab5.log 2>&1
