export CE_PDL=0 EXPR="bhw(r2),(r1)(r2)hw->bhw(r1)|hw" DIMS="[[128,14,14,229],[229,229,3,3]]"
for d in 512 513 514 515; do echo "== EXTRA_DBG=$d"; EXTRA_DBG=$d timeout 60 python tools/tc_phases.py 2>&1 | grep -E "epi_first|end  |first_stage|producer |mma "; done > gpurun_out/exp17.txt 2>&1
