# phase stamps of the TC launches given as arguments of one cfg2 layer (TC_DEBUG build in build_alt)
#   bash tools/phases_one.sh tk 0.1 2 7
kind=$1; cr=$2; shift 2
for n in "$@"; do
  echo "=== $kind$cr TC launch $n"
  CE_LIB_PATH=build_alt/libce.so CE_TC_DBG=544 CE_TC_DBG_AT=$n timeout 120 python tools/tc_phases_layer.py $kind $cr 2>&1 | head -40
done
