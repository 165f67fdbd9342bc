for v in "CE_TC_DBG=64" "CE_TC_DBG=128" "CE_TC_DBG=128 CE_PDL=0"; do
  echo "$v: $(env $v python bench.py --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d.get("layer_fwd_bwd_ms"))')"
done > gpurun_out/exp8.txt 2>&1
