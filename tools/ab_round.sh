timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/t_all.txt 2>&1
for i in 1 2; do
python bench.py --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', d['ms_per_step'], d['e2e']['value'])" >> gpurun_out/ab_bench.txt
CE_PERM_BLOCK=0 CE_EXPAND=0 CE_PAD_PAIR=0 python bench.py --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['ms_per_step'], d['e2e']['value'])" >> gpurun_out/ab_bench.txt
done
for a in "rtr 4,4,8 4,4,4 3 28 256 0.1" "rtr 4,4,4 1,1,3 7 112 256 0.1" "cp 64 3 7 112 128 0.1"; do
  echo "== $a"; timeout 300 python tools/prof_layer.py $a | grep -E " us |total"
  echo "-- old"; CE_PERM_BLOCK=0 CE_EXPAND=0 CE_PAD_PAIR=0 timeout 300 python tools/prof_layer.py $a | grep -E "total"
done > gpurun_out/ab_layers.txt 2>&1
