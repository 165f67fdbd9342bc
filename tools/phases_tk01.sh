for n in 0 1 2 3 4 5 6 7 8; do
  echo "=== tk0.1 TC launch $n"
  CE_LIB_PATH=build_alt/libce.so CE_TC_DBG=544 CE_TC_DBG_AT=$n timeout 120 python tools/tc_phases_layer.py tk 0.1 2>&1 | head -40
done
