export CE_PDL=0
{
for at in 1 0 2; do echo "== tk1.0 launch $at"; CE_TC_DBG=32 CE_TC_DBG_AT=$at timeout 60 python tools/tc_phases_layer.py tk 1.0 2>&1 | tail -11 | cut -c1-200; done
} > gpurun_out/exp33.txt 2>&1
unset CE_PDL
{
for at in 1 0 2; do echo "== PDL tk1.0 launch $at"; CE_TC_DBG=32 CE_TC_DBG_AT=$at timeout 60 python tools/tc_phases_layer.py tk 1.0 2>&1 | tail -11 | cut -c1-200; done
} >> gpurun_out/exp33.txt 2>&1
