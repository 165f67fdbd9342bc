# Several executor knobs A/B'd against the default on one box: bench.py step time, interleaved
# N rounds (default 3).   bash tools/ab_multi.sh N "CE_X=1" "CE_Y=0 CE_Z=1" ...
set -u
N="$1"; shift
for i in $(seq "$N"); do
  for envs in "" "$@"; do
    ms=$(env $envs python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-cfg3 2>/dev/null | tail -1 |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['layer_fwd_bwd_ms'])")
    echo "[${envs:-default}] $ms"
  done
done
