timeout 300 python tools/prof_layer.py tr 256 256 3 14 128 0.3 > gpurun_out/tr.txt 2>&1
