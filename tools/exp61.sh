timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/kernels_$i.json > gpurun_out/bench_$i.txt 2>&1; done
CE_TC_WIDE=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/kernels_nowide.json > gpurun_out/bench_nowide.txt 2>&1
