for L in "tk 1.0" "tt 1.0" "tk 0.1" "tt 0.1"; do TAG="$L" timeout 120 python tools/tc_timing.py $L 2>&1 | grep -E " tc |total"; done > gpurun_out/exp16.txt 2>&1
for v in "CE_TC_PAIR=1" "CE_TC_PAIR=0"; do echo "$v $(env $v timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-250)"; done >> gpurun_out/exp16.txt
