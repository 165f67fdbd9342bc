export CE_PDL=0 CE_TC_MCAST=0 EXPR="bhw(r2),(r1)(r2)hw->bhw(r1)|hw" DIMS="[[128,14,14,229],[229,229,3,3]]"
for d in 531 512; do echo "== EXTRA_DBG=$d"; EXTRA_DBG=$d python tools/tc_phases.py 2>&1 | grep -E "epi_first|end  |first_stage|producer |mma "; done > gpurun_out/exp12.txt 2>&1
