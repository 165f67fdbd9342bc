timeout 600 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/kernels.json > gpurun_out/bench.txt 2>&1
