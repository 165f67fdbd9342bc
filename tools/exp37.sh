timeout 1500 python tools/bench_configs.py --out gpurun_out/configs_r01.json > gpurun_out/configs.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
NCU="ncu --set full --import-source on --clock-control none -k regex:ce_tc_kernel --launch-count 1"
timeout 600 $NCU --launch-skip 1 -o gpurun_out/r01b_tk10_node1 python tools/run_layer.py tk 1.0 1 > gpurun_out/ncu1.log 2>&1
timeout 600 $NCU --launch-skip 4 -o gpurun_out/r01b_tt10_grad6 python tools/run_layer.py tt 1.0 1 > gpurun_out/ncu2.log 2>&1
