export CE_PDL=0
{ for d in 544 552; do echo "== tr0.3 launch 1 dbg $d"; CE_TC_DBG=$d CE_TC_DBG_AT=1 timeout 60 python tools/tc_phases_layer.py tr 0.3 2>&1 | tail -11 | cut -c1-600; done; } > gpurun_out/exp54.txt 2>&1
