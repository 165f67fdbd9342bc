export CE_PDL=0
{
for d in 544 2592 4640 6688; do echo "== tk1.0 launch 1 dbg $d"; CE_TC_DBG=$d CE_TC_DBG_AT=1 timeout 60 python tools/tc_phases_layer.py tk 1.0 2>&1 | tail -11 | cut -c1-200; done
for d in 544 2592 4640; do echo "== tk1.0 launch 6 dbg $d"; CE_TC_DBG=$d CE_TC_DBG_AT=6 timeout 60 python tools/tc_phases_layer.py tk 1.0 2>&1 | tail -11 | cut -c1-200; done
} > gpurun_out/exp31.txt 2>&1
