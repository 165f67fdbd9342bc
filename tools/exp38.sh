{
timeout 120 python tools/prof_layer.py cp 256 256 3 14 128 0.5
timeout 300 python tools/prof_layer.py rtr 4,4,8 4,4,4 3 28 256 0.1
timeout 300 python tools/prof_layer.py rtr 4,4,4 1,1,3 7 112 256 0.1
timeout 300 python tools/prof_layer.py cp 64 3 7 112 128 1.0
} > gpurun_out/exp38.txt 2>&1
