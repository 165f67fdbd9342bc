timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python tools/prof_layer.py tr 256 256 3 14 128 0.3 > gpurun_out/tr.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$i.txt 2>&1; done
CE_TC_CONTIG=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nocontig.txt 2>&1
