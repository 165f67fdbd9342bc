timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/exp18.txt
for v in "CE_CONCURRENT=1" "CE_CONCURRENT=0"; do echo "$v $(env $v timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-200)"; done >> gpurun_out/exp18.txt
