set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_tc_kat.py -x -q 2>&1 | tail -30 > gpurun_out/kat.txt
cat gpurun_out/kat.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_native.json 2> gpurun_out/bench_native.err
CE_TC_NATIVE_MN=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_xpose.json 2> gpurun_out/bench_xpose.err
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_native2.json 2>> gpurun_out/bench_native.err
for f in gpurun_out/bench_*.json; do python -c "import json,sys; j=json.load(open('$f')); print('$f', j['ms_per_step'], j['value'], j['layer_fwd_bwd_ms'])"; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/gputests.txt
cat gpurun_out/gputests.txt
