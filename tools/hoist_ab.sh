# A/B of layout hoisting (CE_HOIST) on the cfg3 RTR 64->128 layer and the cfg3 stack
for h in 0 1; do echo "=== HOIST $h"; CE_HOIST=$h timeout 300 python tools/prof_layer.py rtr 4,4,8 4,4,4 3 28 256 0.1 | grep -v "^fwd\|^bwd"; done > gpurun_out/hoist_64_128.txt 2>&1
CE_HOIST=1 timeout 600 python tools/bench_configs.py --only cfg3 --out gpurun_out/cfg3_h1.json > gpurun_out/cfg3_h1.log 2>&1
