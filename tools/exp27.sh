export CE_PDL=0
run() { echo "== $1 $2 dbg=$3"; EXPR="$1" DIMS="$2" EXTRA_DBG=$3 timeout 60 python tools/tc_phases.py 2>&1 | tail -11; }
{
run "abw,bs->aws" "[[273,273,3],[273,256]]" 512
run "at,abh->tbh" "[[273,256],[273,273,3]]" 512
run "bhwc,chw->bhw" "[[128,14,14,57],[57,14,14]]" 0
run "bhwr,bhws->rs" "[[128,14,14,57],[128,14,14,64]]" 512
} > gpurun_out/exp27.txt 2>&1
