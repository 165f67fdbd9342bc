timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python tools/prof_layer.py cp 64 3 7 112 128 1.0 > gpurun_out/cp1.txt 2>&1
