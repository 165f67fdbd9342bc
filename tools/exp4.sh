C='[("bhws,rs->bhwr",[[128,14,14,256],[57,256]]),("bhws,rs->bhwr",[[1,14,14,256],[57,256]]),("bshw,rs->bhwr",[[128,256,14,14],[229,256]])]'
for c in 0 1; do CE_CARVEOUT=$c TAG=co$c CASES="$C" python tools/tc_micro.py; done > gpurun_out/micro4.txt 2>&1
for c in 0 1; do CE_CARVEOUT=$c python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-300; done >> gpurun_out/micro4.txt
