for e in "CE_TC_TAIL=0" "CE_TC_CTMA=0" "CE_TC_LEAN=0" ""; do
  echo "== $e"
  env $e timeout 300 python -m pytest "tests/test_gpu_parity.py::test_baseline_layers_full_size" -m gpu -x -q -k "auto" 2>&1 | tail -3
done
