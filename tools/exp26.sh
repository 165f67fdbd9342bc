export CE_PDL=0 EXPR="bshw,rs->bhwr" DIMS="[[128,256,14,14],[57,256]]"
for d in 0 1 8 8192 4096 2048 9 512; do echo "== EXTRA_DBG=$d"; EXTRA_DBG=$d timeout 60 python tools/tc_phases.py 2>&1 | grep -vE "^\s*$" | tail -12; done > gpurun_out/exp26.txt 2>&1
export EXPR="bhws,rs->bhwr" DIMS="[[128,14,14,256],[57,256]]"
for d in 0 512; do echo "== KMAJ EXTRA_DBG=$d"; EXTRA_DBG=$d timeout 60 python tools/tc_phases.py 2>&1 | tail -12; done >> gpurun_out/exp26.txt 2>&1
