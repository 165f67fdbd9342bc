C='[("bhws,rs->bhwr",[[1,14,14,256],[57,256]])]'
CASES="$C" ncu --set full --import-source on --clock-control none -k regex:ce_tc_kernel -s 3 -c 1 -o gpurun_out/tiny python tools/tc_micro.py > gpurun_out/ncu5.log 2>&1
C='[("bhws,rs->bhwr",[[128,14,14,256],[57,256]])]'
CASES="$C" ncu --set full --import-source on --clock-control none -k regex:ce_tc_kernel -s 3 -c 1 -o gpurun_out/kmaj57 python tools/tc_micro.py >> gpurun_out/ncu5.log 2>&1
