timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "layer_scores or scores_parity or pearson" > gpurun_out/t17.log 2>&1; echo t17=$? > gpurun_out/rc16.txt
