for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$i.txt 2>&1; done
