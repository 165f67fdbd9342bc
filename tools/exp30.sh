export CE_PDL=0
timeout 600 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
{
for at in 1 0 2 6; do for d in 544; do echo "== tk1.0 launch $at dbg $d"; CE_TC_DBG=$d CE_TC_DBG_AT=$at timeout 60 python tools/tc_phases_layer.py tk 1.0 2>&1 | tail -11 | cut -c1-300; done; done
} > gpurun_out/exp30.txt 2>&1
unset CE_PDL
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --profile-json gpurun_out/kernels.json > gpurun_out/bench.txt 2>&1
