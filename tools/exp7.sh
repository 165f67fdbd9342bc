bash tools/exp6.sh
CE_TC_DBG=0 python tools/tc_micro.py > gpurun_out/micro7.txt 2>&1
python -m pytest tests -m gpu -q -x 2>&1 | tail -2 >> gpurun_out/micro7.txt
python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | cut -c1-250 >> gpurun_out/micro7.txt
