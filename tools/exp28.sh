export CE_PDL=0
{
for at in 6 5 1; do for d in 544 545 8736; do echo "== tk1.0 launch $at dbg $d"; CE_TC_DBG=$d CE_TC_DBG_AT=$at timeout 60 python tools/tc_phases_layer.py tk 1.0 2>&1 | tail -11; done; done
} > gpurun_out/exp28.txt 2>&1
