export CE_PDL=0 EXPR="(r1)t,(r1)(r2)h->ht(r2)" DIMS="[[273,256],[273,273,3]]"
for d in 512; do echo "== EXTRA_DBG=$d"; EXTRA_DBG=$d timeout 60 python tools/tc_phases.py 2>&1 | grep -E "epi_|end  |first_stage|producer|mma"; done > gpurun_out/exp19.txt 2>&1
CASES='[("(r1)t,(r1)(r2)h->ht(r2)",[[273,256],[273,273,3]])]' timeout 60 python tools/tc_micro.py >> gpurun_out/exp19.txt 2>&1
CE_TC_PAIR=0 CASES='[("(r1)t,(r1)(r2)h->ht(r2)",[[273,256],[273,273,3]])]' timeout 60 python tools/tc_micro.py >> gpurun_out/exp19.txt 2>&1
