export EXPR="bhws,rs->bhwr" DIMS="[[128,14,14,256],[57,256]]"
for d in 0 2 6 15; do echo "== EXTRA_DBG=$d"; EXTRA_DBG=$d python tools/tc_phases.py; done > gpurun_out/phases.txt 2>&1
export DIMS="[[8,14,14,256],[57,256]]"
for d in 0 15; do echo "== small EXTRA_DBG=$d"; EXTRA_DBG=$d python tools/tc_phases.py; done >> gpurun_out/phases.txt 2>&1
CASES='[("bhws,rs->bhwr",[[8,14,14,256],[57,256]]),("bhws,rs->bhwr",[[1,14,14,256],[57,256]])]' python tools/tc_micro.py >> gpurun_out/phases.txt 2>&1
