timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/exp20.txt
for L in "tk 1.0" "tt 1.0" "tk 0.1" "tt 0.1"; do TAG="$L" timeout 120 python tools/tc_timing.py $L 2>&1 | grep -E " tc |permute|total"; done >> gpurun_out/exp20.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/exp20.txt
