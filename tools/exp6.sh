export EXPR="bhws,rs->bhwr" DIMS="[[1,14,14,256],[57,256]]"
for d in 0 15; do echo "== tiny EXTRA_DBG=$d"; EXTRA_DBG=$d python tools/tc_phases.py; done > gpurun_out/phases6.txt 2>&1
export DIMS="[[128,14,14,256],[57,256]]"
for d in 0; do echo "== big EXTRA_DBG=$d"; EXTRA_DBG=$d python tools/tc_phases.py; done >> gpurun_out/phases6.txt 2>&1
