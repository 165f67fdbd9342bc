# A/B of the tiny-K stream-kernel rule bound (CE_TINYK) on cfg3 conv1, 64->128 and the cfg3 stack
for t in 8 16 36; do echo "=== TINYK $t"; CE_TINYK=$t timeout 300 python tools/prof_layer.py rtr 4,4,4 1,1,3 7 112 256 0.1 | grep -v "^fwd\|^bwd"; done > gpurun_out/tinyk_conv1.txt 2>&1
for t in 8 16 36; do echo "=== TINYK $t"; CE_TINYK=$t timeout 300 python tools/prof_layer.py rtr 4,4,8 4,4,4 3 28 256 0.1 | grep -v "^fwd\|^bwd"; done > gpurun_out/tinyk_64_128.txt 2>&1
for t in 16 36; do CE_TINYK=$t timeout 600 python tools/bench_configs.py --only cfg3 --out gpurun_out/cfg3_tk$t.json > /dev/null 2>&1; done
