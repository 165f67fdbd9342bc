python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/exp14.txt
for L in "tk 1.0" "tt 1.0" "tt 0.1"; do TAG="$L" python tools/tc_timing.py $L 2>&1 | grep -E "permute|total"; done >> gpurun_out/exp14.txt 2>&1
python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-250 >> gpurun_out/exp14.txt
