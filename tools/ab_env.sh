# A/B an executor knob on one box: bench.py step time with and without the environment
# settings given as arguments, interleaved N times (default 3), then per-kernel device times
# of the cfg2 layers (prof_layer.py) both ways.
#   bash tools/ab_env.sh "CE_TC_QSPLIT=1" [N]
set -u
ENVS="$1"; N="${2:-3}"
for i in $(seq "$N"); do
  for side in on off; do
    if [ "$side" = on ]; then pre="env $ENVS"; else pre="env"; fi
    $pre python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$side', d['ms_per_step'])"
  done
done
for a in "tk 256 256 3 14 128 0.1" "tk 256 256 3 14 128 1.0" "tt 256 256 3 14 128 0.1" "tt 256 256 3 14 128 1.0"; do
  echo "== $a"
  env $ENVS python tools/prof_layer.py $a | grep -E " us |total" > /tmp/ab_on.txt
  python tools/prof_layer.py $a | grep -E " us |total" > /tmp/ab_off.txt
  python - <<'PY'
on = [l.split() for l in open('/tmp/ab_on.txt')]
off = [l.split() for l in open('/tmp/ab_off.txt')]
for a, b in zip(off, on):
    t = (lambda r: r[1] if r[0] == 'total' else r[2])
    print(f"{a[0]:16s} off {t(a):>10s}  on {t(b):>10s}")
PY
done
