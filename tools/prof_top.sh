# ncu --set full captures of the top TC kernels (one launch each) + bench with pipelined e2e
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/kernels.json > gpurun_out/bench.txt 2>&1
NCU="ncu --set full --import-source on --clock-control none -k regex:ce_tc_kernel --launch-count 1"
timeout 600 $NCU --launch-skip 1 -o gpurun_out/tk10_node1 python tools/run_layer.py tk 1.0 1 > gpurun_out/ncu1.log 2>&1
timeout 600 $NCU --launch-skip 6 -o gpurun_out/tk10_grad3 python tools/run_layer.py tk 1.0 1 > gpurun_out/ncu2.log 2>&1
timeout 600 $NCU --launch-skip 0 -o gpurun_out/tk01_node0 python tools/run_layer.py tk 0.1 1 > gpurun_out/ncu3.log 2>&1
