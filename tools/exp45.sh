ncu --set full --clock-control none -k regex:ce_stream_kernel --launch-count 1 -o gpurun_out/cp_dw python tools/prof_layer.py cp 256 256 3 14 128 0.5 > gpurun_out/ncu_cp.log 2>&1
