timeout 600 python -m pytest tests/test_tc_kat.py -q 2>&1 | tail -4
for i in 1 2; do
for cfg in "CE_X=0" "CE_TC_NATIVE_MN=0" "CE_MN_REPACK=2" "CE_MN_REPACK=0"; do
  env $cfg timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err || tail -5 /tmp/b.err
  python -c "import json; j=json.load(open('/tmp/b.json')); print('$cfg', j['ms_per_step'], j['value'], j['layer_fwd_bwd_ms'])"
done
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
