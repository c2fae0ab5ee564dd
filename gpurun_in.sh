timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_checked.py -x -q -m gpu -k "quantize or edge or checked or guard or config" > gpurun_out/t16.log 2>&1; echo t16=$? > gpurun_out/rc14.txt
timeout 600 python tools/quant_ab.py --layers 8 --rounds 5 prod qold > gpurun_out/qab5.log 2>&1
timeout 600 python tools/quant_ab.py --cfg C2 --layers 12 --rounds 5 prod qold >> gpurun_out/qab5.log 2>&1
for s in 16 32 64 128; do timeout 600 python tools/quant_ab.py --cfg C4-$s --layers 3 --rounds 4 prod qold >> gpurun_out/qab5.log 2>&1; done
