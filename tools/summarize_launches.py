"""Summarise an ncu launch list of bench.py (tools/round_artifacts.sh) for profiles/.

  python tools/summarize_launches.py gpurun_out/launches.csv > profiles/ncu_launches_r01_summary.txt

One timed step = the launches between the first two L2-flush fills (torch elementwise
kernels) that bracket a cfg2 step; per kernel template: launches, summed duration, share,
DRAM bytes.  Durations are ncu's serialised, cold-cache replays.
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    ids = {}
    for r in rows[1:]:
        i = int(r[0])
        d = ids.setdefault(i, {"name": r[4].split("(")[0].replace("<unnamed>::", "").replace("void ", ""),
                               "grid": r[8]})
        d[r[12]] = float(r[14].replace(",", ""))
    order = sorted(ids)
    flush = [i for i in order if "elementwise" in ids[i]["name"] or "at::" in ids[i]["name"]]
    # the first pair of flush fills with a step between them (other torch fills, e.g. the
    # warm-up's output buffers, sit back to back)
    k = next(j for j in range(len(flush) - 1) if flush[j + 1] - flush[j] > 20)
    lo, hi = flush[k] + 1, flush[k + 1] - 1
    step = [i for i in order if lo <= i <= hi]
    tot = sum(ids[i]["gpu__time_duration.sum"] for i in step) / 1e3
    longest = max(step, key=lambda i: ids[i]["gpu__time_duration.sum"])
    print(f"One timed cfg2 step (launch IDs {lo}..{hi} of {path.split('/')[-1]}; serialised replay, cold caches):")
    print(f"{len(step)} kernels, {tot:.1f} us summed (the device-timed step with concurrency and PDL is shorter)")
    lt = ids[longest]["gpu__time_duration.sum"] / 1e3
    print(f"longest launch: {ids[longest]['name']} grid {ids[longest]['grid']} {lt:.1f} us = {lt / tot:.3f} of the step")
    print()
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for i in step:
        a = agg[ids[i]["name"]]
        a[0] += 1
        a[1] += ids[i]["gpu__time_duration.sum"] / 1e3
        a[2] += (ids[i].get("dram__bytes_read.sum", 0) + ids[i].get("dram__bytes_write.sum", 0)) / 1e6
    print("kernel, launches, total us, share, DRAM MB (read+write)")
    for name, (n, us, mb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name}, {n}, {us:.1f}, {us / tot:.3f}, {mb:.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
