export CE_PDL=0 EXPR="bshw,rs->bhwr" DIMS="[[128,256,14,14],[57,256]]"
for d in 512 2560 4608 6658; do echo "== EXTRA_DBG=$d"; EXTRA_DBG=$d timeout 60 python tools/tc_phases.py 2>&1 | grep -E "epi_first|first_stage|producer|mma "; done > gpurun_out/exp23.txt 2>&1
