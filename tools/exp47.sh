for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$i.txt 2>&1; done
timeout 1500 python tools/bench_configs.py --out gpurun_out/configs_r01.json > gpurun_out/configs.log 2>&1
timeout 300 python tools/prof_layer.py rtr 4,4,8 4,4,4 3 28 256 0.1 > gpurun_out/rtr.txt 2>&1
