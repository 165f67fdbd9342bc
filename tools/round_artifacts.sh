# Round artifacts on one B200: GPU tests, smoke, bench x3 (ours) + reference arm, ncu launch
# list of one bench step, ncu --set full of the top tensor-core launches and of one launch per
# SIMT / permute / fused family, every BASELINE config (tools/bench_configs.py).
# Summaries: python tools/summarize_launches.py / summarize_ncu_full.py / summarize_families.py
set -x
TAG=${TAG:-r02}
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/smoke.txt
for i in 1 2 3; do timeout 900 python bench.py --steps 10 --warmup 3 --profile-json gpurun_out/kernels_$i.json > gpurun_out/bench_$i.txt 2>&1; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-cfg3 > gpurun_out/ncu_bench.log 2>&1
NCU="ncu --set full --import-source on --clock-control none -k regex:ce_tc_kernel --launch-count 1"
timeout 600 $NCU --launch-skip 1 -o gpurun_out/full_tk10_node1 python tools/run_layer.py tk 1.0 1 > gpurun_out/ncu1.log 2>&1
timeout 600 $NCU --launch-skip 5 -o gpurun_out/full_tk10_grad4 python tools/run_layer.py tk 1.0 1 > gpurun_out/ncu2.log 2>&1
timeout 600 $NCU --launch-skip 6 -o gpurun_out/full_tk10_grad3 python tools/run_layer.py tk 1.0 1 > gpurun_out/ncu3.log 2>&1
timeout 600 $NCU --launch-skip 4 -o gpurun_out/full_tt10_grad6 python tools/run_layer.py tt 1.0 1 > gpurun_out/ncu4.log 2>&1
timeout 600 $NCU --launch-skip 1 -o gpurun_out/full_tt10_node1 python tools/run_layer.py tt 1.0 1 > gpurun_out/ncu5.log 2>&1
bash tools/ncu_families.sh
timeout 1800 python tools/bench_configs.py --out gpurun_out/configs_$TAG.json > gpurun_out/configs.log 2>&1
# summaries on the box (the .ncu-rep files can exceed gpurun's 64 MiB copy-back limit)
mkdir -p gpurun_out/prof
python tools/summarize_launches.py gpurun_out/launches.csv > gpurun_out/prof/ncu_launches_${TAG}_summary.txt 2>&1
cp gpurun_out/launches.csv gpurun_out/prof/ncu_launches_${TAG}.csv
python tools/summarize_ncu_full.py gpurun_out gpurun_out/prof $TAG > gpurun_out/prof/summarize_full.log 2>&1
python tools/summarize_families.py gpurun_out gpurun_out/prof $TAG > gpurun_out/prof/summarize_families.log 2>&1
du -sh gpurun_out/*.ncu-rep > gpurun_out/prof/rep_sizes.txt 2>&1
rm -f gpurun_out/*.ncu-rep
