export CE_PDL=0 EXPR="bhw(r2),(r1)(r2)hw->bhw(r1)|hw" DIMS="[[128,14,14,229],[229,229,3,3]]"
for d in 0 1 2 3 15; do echo "== tk1.0 node1 EXTRA_DBG=$d"; EXTRA_DBG=$d python tools/tc_phases.py 2>&1 | grep -v "Exception\|Traceback\|File\|TypeError"; done > gpurun_out/exp9.txt 2>&1
