timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -8 > gpurun_out/exp25.txt
