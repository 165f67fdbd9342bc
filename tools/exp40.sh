timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
{
timeout 300 python tools/prof_layer.py rtr 4,4,8 4,4,4 3 28 256 0.1
timeout 300 python tools/prof_layer.py rtr 4,4,4 1,1,3 7 112 256 0.1
} > gpurun_out/exp40.txt 2>&1
