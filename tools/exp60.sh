export CE_PDL=0
CE_TC_DBG=544 CE_TC_DBG_AT=1 timeout 60 python tools/tc_phases_layer.py tr 0.3 > gpurun_out/exp60.txt 2>&1
