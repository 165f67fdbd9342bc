timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_base_$i.txt 2>&1; done
for i in 1 2; do CE_REPACK_MN=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/kernels_rmn.json > gpurun_out/bench_rmn_$i.txt 2>&1; done
