for cfg in "" "CE_TC_MN_SBO=1024" "CE_TC_MN_LBO=512 CE_TC_MN_SBO=4096" "CE_TC_MN_TMASWZ=5" "CE_TC_MN_LAYOUT=2 CE_TC_MN_TMASWZ=3 CE_TC_MN_SBO=1024" "CE_TC_MN_LAYOUT=1 CE_TC_MN_TMASWZ=3 CE_TC_MN_SBO=1024"; do
  env $cfg timeout 120 python tools/mn_probe.py 2>&1 | tail -6
done
