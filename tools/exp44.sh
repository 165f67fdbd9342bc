timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
{
for at in 1 2; do echo "== PDL tk1.0 launch $at"; CE_TC_DBG=32 CE_TC_DBG_AT=$at timeout 60 python tools/tc_phases_layer.py tk 1.0 2>&1 | tail -11 | cut -c1-200; done
} > gpurun_out/exp44.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/kernels_$i.json > gpurun_out/bench_$i.txt 2>&1; done
CE_TC_SK=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nosk.txt 2>&1
