export CE_PDL=0 EXPR="bshw,rs->bhwr" DIMS="[[128,256,14,14],[57,256]]"
for d in 512; do echo "== EXTRA_DBG=$d"; EXTRA_DBG=$d timeout 60 python tools/tc_phases.py 2>&1 | grep -E "epi_|end  |first_stage|setup|producer|mma"; done > gpurun_out/exp21.txt 2>&1
unset CE_PDL EXPR DIMS
for v in "CE_TC_DBG=64" "CE_TC_DBG=128"; do echo "$v $(env $v timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | cut -c180-240)"; done >> gpurun_out/exp21.txt
