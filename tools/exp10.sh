export CE_PDL=0 EXPR="bhw(r2),(r1)(r2)hw->bhw(r1)|hw" DIMS="[[128,14,14,229],[229,229,3,3]]"
for v in "CE_TC_MCAST=0" "CE_TC_NCAP=128" "CE_TC_NCAP=128 CE_TC_MCAST=0" "CE_TC_NCAP=64"; do
for d in 0 3; do echo "== $v EXTRA_DBG=$d"; env $v EXTRA_DBG=$d python tools/tc_phases.py 2>&1 | grep -E "epi_first|end  |first_stage"; done; done > gpurun_out/exp10.txt 2>&1
