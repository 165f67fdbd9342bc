export CE_PDL=0 EXPR="bshw,rs->bhwr" DIMS="[[128,256,14,14],[57,256]]"
for d in 6658 14850 23042 31234 6659 31235; do echo "== EXTRA_DBG=$d"; EXTRA_DBG=$d timeout 60 python tools/tc_phases.py 2>&1 | grep -E "producer|mma "; done > gpurun_out/exp24.txt 2>&1
export EXPR="bhws,rs->bhwr" DIMS="[[128,14,14,256],[57,256]]"
for d in 6658 6659; do echo "== KMAJ EXTRA_DBG=$d"; EXTRA_DBG=$d timeout 60 python tools/tc_phases.py 2>&1 | grep -E "producer|mma "; done >> gpurun_out/exp24.txt 2>&1
