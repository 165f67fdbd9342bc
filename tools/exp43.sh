{
for k in "tk 1.0" "tt 1.0" "tt 0.1"; do echo "== $k"; CE_TIMELINE=1 timeout 120 python tools/tc_timing.py $k 2>&1 | grep -E "timeline|total"; done
} > gpurun_out/exp43.txt 2>&1
