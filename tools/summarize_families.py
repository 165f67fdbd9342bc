"""Summarise the per-family ncu captures of tools/ncu_families.sh into profiles/:
ncu_families_<tag>.json and .md -- duration, DRAM bytes, achieved HBM GB/s and its fraction
of the measured copy bandwidth (MEASURED_PEAKS.json), occupancy, registers.

  python tools/summarize_families.py gpurun_out profiles r02
"""
import csv
import io
import json
import os
import subprocess
import sys

CAPTURES = {
    "full_cp10_stencil": ("stencil (ce_dw_kernel)", "CP conv2_x 64->64 @56 B128 cr1.0 (R=275), depthwise h-step"),
    "full_cp10_dwgrad": ("depthwise filter grad (ce_dwgrad_kernel)", "same layer, dF_w"),
    "full_cp01_dw2": ("fused h+w stencil pair (ce_dw2_kernel, F1)", "CP conv2_x cr0.1 (R=27), forward pair"),
    "full_tk10_permute": ("permute (ce_transpose_kernel)", "cfg2 TK cr1.0, first transpose launch"),
    "full_cp_conv1_stream": ("stream, tiny K (ce_stream_blk_kernel)", "CP conv1 3->64 @112 B32 cr1.0, node0 (K=3)"),
    "full_rtr_conv1_pconv": ("plane conv (ce_pconv_kernel)", "cfg3 RTR conv1 3->64 @112 B256, X * W4 (7x7, 9 channels)"),
    "full_rtr_conv1_pconv_wgrad": ("plane-conv filter grad (ce_pconv_wgrad_kernel)", "same layer, dW4"),
}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "lts__t_sector_hit_rate.pct", "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    return {k: (v[h.index(k)], units[h.index(k)]) for k in h if k in METRICS or k == "Kernel Name"}


def to_num(val, unit):
    x = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3}
    return x * scale.get(unit, 1)


def main(src, dst, tag):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        peak = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6550.0
    res = {"source": "ncu --set full --clock-control none, one launch each (tools/ncu_families.sh), B200",
           "hbm_peak_gbs": peak, "kernels": {}}
    lines = [f"# ncu per kernel family ({tag})", "", f"HBM peak (MEASURED_PEAKS.json copy bandwidth): {peak} GB/s", "",
             "| family | workload | us | DRAM MB (r+w) | GB/s | of peak | warps active | regs |",
             "|---|---|---|---|---|---|---|---|"]
    for name, (fam, wl) in CAPTURES.items():
        rep = os.path.join(src, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        m = raw(rep)
        us = to_num(*m["gpu__time_duration.sum"])
        mb = (to_num(*m["dram__bytes_read.sum"]) + to_num(*m["dram__bytes_write.sum"])) / 1e6
        gbs = mb * 1e6 / (us * 1e-6) / 1e9
        res["kernels"][name] = {"family": fam, "workload": wl, "kernel": m["Kernel Name"][0].strip(), "us": us,
                                "dram_mb": round(mb, 3), "gbs": round(gbs, 1), "frac_of_hbm_peak": round(gbs / peak, 3),
                                "warps_active_pct": float(m["sm__warps_active.avg.pct_of_peak_sustained_active"][0]),
                                "registers": int(m["launch__registers_per_thread"][0])}
        r = res["kernels"][name]
        lines.append(f"| {fam} | {wl} | {us:.1f} | {mb:.1f} | {gbs:.0f} | {gbs / peak:.2f} | "
                     f"{r['warps_active_pct']:.0f}% | {r['registers']} |")
    json.dump(res, open(os.path.join(dst, f"ncu_families_{tag}.json"), "w"), indent=1)
    open(os.path.join(dst, f"ncu_families_{tag}.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
