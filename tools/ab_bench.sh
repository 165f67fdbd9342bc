# bench.py A/B: current defaults vs the knobs of this session's RTR work turned off
for i in 1 2 3; do
python bench.py --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', d['ms_per_step'], d['e2e']['value'])"
CE_PERM_BLOCK=0 CE_EXPAND=0 CE_PAD_PAIR=0 CE_PACK_FIRST=1 python bench.py --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['ms_per_step'], d['e2e']['value'])"
done
