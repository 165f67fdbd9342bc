# ncu --set full (with source) of the store-bound RTR 64->128 node0 launch (the 5.1 GB
# rank-pair intermediate written in 128x100 tiles), summarised for profiles/: raw metrics,
# details, and the top SASS stall sites (DESIGN §10 item 2).
mkdir -p gpurun_out/rtrst
R='python tools/prof_layer.py rtr 4,4,8 4,4,4 3 28 256 0.1'
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ce_tc_kernel -c 1 -o gpurun_out/rtrst/rtr_node0 $R > gpurun_out/rtrst/ncu.log 2>&1
ncu -i gpurun_out/rtrst/rtr_node0.ncu-rep --page raw --csv > gpurun_out/rtrst/ncu_rtr64_node0_r02_raw.csv 2>&1
ncu -i gpurun_out/rtrst/rtr_node0.ncu-rep --page details --csv > gpurun_out/rtrst/ncu_rtr64_node0_r02_details.csv 2>&1
ncu -i gpurun_out/rtrst/rtr_node0.ncu-rep --page source --csv --print-source sass > gpurun_out/rtrst/sass.csv 2>&1
python - <<'PY' > gpurun_out/rtrst/ncu_rtr64_node0_r02_stalls.txt
import csv
rows = list(csv.reader(open("gpurun_out/rtrst/sass.csv")))
h = rows[1]; data = rows[2:]
si = h.index("Source"); wi = h.index("Warp Stall Sampling (All Samples)"); ei = h.index("Instructions Executed")
tot = sum(int(r[wi]) for r in data if len(r) > wi and r[wi].isdigit())
print("RTR 64->128 node0 (ce_tc_kernel LEAN 128): top SASS stall sites, share of all warp-stall samples")
print("(the BSYNC after DEPBAR.LE SB0 is the epilogue lanes waiting on lane 0's cp.async.bulk.wait_group.read)")
for i, r in sorted(((i, r) for i, r in enumerate(data) if len(r) > wi and r[wi].isdigit()), key=lambda x: -int(x[1][wi]))[:15]:
    prev = data[i - 1][si].strip() if i else ""
    print(f"{int(r[wi]) / tot:6.3f}  #{i:5d}  {r[si].strip()[:60]:60s}  exec={r[ei]}  prev: {prev[:40]}")
PY
rm -f gpurun_out/rtrst/*.ncu-rep gpurun_out/rtrst/sass.csv
