timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/t_all.txt 2>&1
for i in 1 2 3; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qsplit', d['ms_per_step'])"
CE_TC_QSPLIT=0 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old', d['ms_per_step'])"
done
for a in "tk 256 256 3 14 128 1.0" "tt 256 256 3 14 128 1.0"; do
python tools/prof_layer.py $a | grep -E "^[a-z:0-9A-Z]+ +tc|total" > /tmp/a.txt
CE_TC_QSPLIT=0 python tools/prof_layer.py $a | grep -E "^[a-z:0-9A-Z]+ +tc|total" > /tmp/b.txt
python - <<'PY'
o=[l.split() for l in open('/tmp/b.txt')]; n=[l.split() for l in open('/tmp/a.txt')]
for a,b in zip(o,n): print(f"{a[0]:16s} old {a[2] if a[0]!='total' else a[1]:>10s} new {b[2] if b[0]!='total' else b[1]:>10s}")
PY
done
