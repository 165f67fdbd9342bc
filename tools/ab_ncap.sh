for i in 1 2; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ncap256', d['ms_per_step'])"
CE_TC_NCAP=128 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ncap128', d['ms_per_step'])"
done
for a in "tk 256 256 3 14 128 1.0" "tt 256 256 3 14 128 1.0" "tk 256 256 3 14 128 0.1" "tt 256 256 3 14 128 0.1"; do
  echo "== $a"
  python tools/prof_layer.py $a | grep -E "^[a-z:0-9A-Z]+ +tc|total" > /tmp/a.txt
  CE_TC_NCAP=128 python tools/prof_layer.py $a | grep -E "^[a-z:0-9A-Z]+ +tc|total" > /tmp/b.txt
  python - <<'PY'
o=[l.split() for l in open('/tmp/a.txt')]; n=[l.split() for l in open('/tmp/b.txt')]
for a,b in zip(o,n): print(f"{a[0]:16s} {a[2] if a[0]!='total' else a[1]:>10s} {b[2] if b[0]!='total' else b[1]:>10s}")
PY
done
