for d in 0 1 2 4 6; do CE_TC_DBG=$d python tools/tc_micro.py; done > gpurun_out/micro.txt 2>&1
