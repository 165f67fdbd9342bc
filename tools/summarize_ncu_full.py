"""Turn the `ncu --set full` captures of tools/round_artifacts.sh into profiles/ files:
ncu_<name>_r01_{details,raw}.csv and ncu_traffic_r01.json (DRAM bytes per launch, used by
bench.py's roofline `traffic`).

  python tools/summarize_ncu_full.py gpurun_out profiles
"""
import csv
import io
import json
import os
import subprocess
import sys

CAPTURES = {  # capture file -> step label (tools/run_layer.py layer, executor step)
    "full_tk10_node1": "tk1.0:node1",
    "full_tk10_grad4": "tk1.0:grad:4",
    "full_tk10_grad3": "tk1.0:grad:3",
    "full_tt10_grad6": "tt1.0:grad:6",
    "full_tt10_node1": "tt1.0:node1",
}


def ncu_page(rep, page):
    return subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True,
                          check=True).stdout


def main(src, dst, tag="r02"):
    os.makedirs(dst, exist_ok=True)
    traffic = {"source": "ncu --set full --clock-control none, one launch each (tools/round_artifacts.sh), B200",
               "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch; cold-cache replay", "kernels": {}}
    for cap, label in CAPTURES.items():
        rep = os.path.join(src, cap + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        short = cap.replace("full_", "")
        details = ncu_page(rep, "details")
        raw = ncu_page(rep, "raw")
        open(os.path.join(dst, f"ncu_{short}_{tag}_details.csv"), "w").write(details)
        open(os.path.join(dst, f"ncu_{short}_{tag}_raw.csv"), "w").write(raw)
        rows = list(csv.reader(io.StringIO(raw)))
        h, units, v = rows[0], rows[1], rows[2]

        def m(name, scale=1.0):
            i = h.index(name)
            u = units[i]
            x = float(v[i].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "msecond": 1e3,
                    "nsecond": 1e-3}.get(u, 1)
            return x * mult * scale

        rd, wr = m("dram__bytes_read.sum"), m("dram__bytes_write.sum")
        ent = {"dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
               "duration_us": round(m("gpu__time_duration.sum"), 3), "kernel": v[h.index("Kernel Name")],
               "capture": f"{cap}.ncu-rep (summarised in profiles/ncu_{short}_{tag}_*.csv)"}
        for name, key in [("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_active_pct")]:
            if name in h:
                ent[key] = float(v[h.index(name)].replace(",", ""))
        traffic["kernels"][label] = ent
    with open(os.path.join(dst, f"ncu_traffic_{tag}.json"), "w") as f:
        json.dump(traffic, f, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:4])
