L='python tools/prof_layer.py rtr 4,4,8 4,4,4 3 28 256 0.1'
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ce_tc_kernel --launch-skip 4 -c 1 -o gpurun_out/rtr28_grad6 $L > gpurun_out/ncu_g6.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ce_tc_kernel --launch-skip 8 -c 1 -o gpurun_out/rtr28_grad5 $L > gpurun_out/ncu_g5.log 2>&1
