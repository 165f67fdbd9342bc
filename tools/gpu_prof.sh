# per-kernel device times of the four cfg2 layers (fwd+bwd)
for a in "tk 256 256 3 14 128 0.1" "tk 256 256 3 14 128 1.0" "tt 256 256 3 14 128 0.1" "tt 256 256 3 14 128 1.0"; do
  echo "== $a"; python tools/prof_layer.py $a
done
