# per-step device times of the cfg2 bench layers' permutes, block permute on/off
for a in "tk 256 256 3 14 128 0.1" "tk 256 256 3 14 128 1.0" "tt 256 256 3 14 128 0.1" "tt 256 256 3 14 128 1.0"; do
  echo "== $a"
  python tools/prof_layer.py $a | grep -E " us |total" | grep -E "^[a-z:0-9A-Z]+ +permute|total" > /tmp/new.txt
  CE_PERM_BLOCK=0 python tools/prof_layer.py $a | grep -E " us |total" | grep -E "^[a-z:0-9A-Z]+ +permute|total" > /tmp/old.txt
  python - <<'PY'
o=[l.split() for l in open('/tmp/old.txt')]; n=[l.split() for l in open('/tmp/new.txt')]
for a,b in zip(o,n): print(f"{a[0]:16s} {a[2] if a[0]!='total' else a[1]:>10s} {b[2] if b[0]!='total' else b[1]:>10s}")
PY
done
