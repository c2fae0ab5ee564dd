./tools/bin/ubench_tp > gpurun_out/ubench_tp.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C5 --rounds 6 prod tp tp3 > gpurun_out/ab_c5.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C3 prod tp tp3 > gpurun_out/ab_c3.log 2>&1
timeout 600 python tools/decode_ab.py --cfg C4 --layers 4 prod tp tp3 > gpurun_out/ab_c4.log 2>&1
WQ_VARIANT=tp3 timeout 600 python tools/decode_err.py C1 C2 C3 C5 > gpurun_out/err_tp.log 2>&1
