"""Per-step device times of single pairwise problems (TC kernel experiments).
usage: CE_TC_DBG=<flags> python tools/tc_micro.py  [cases from CASES env, python literal list of (expr, dims)]
Needs the debug build of the TC kernel (flags and stamps are compiled out otherwise):
  rm -rf build && make -C paper_2401_03384_b200/csrc TC_DEBUG=1   (rebuild normally afterwards)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_03384_b200 as ce  # noqa: E402
from paper_2401_03384_b200.device import Context, Executor  # noqa: E402

DEFAULT = [
    ("bshw,rs->bhwr", [[128, 256, 14, 14], [57, 256]]),   # MN-major A, skinny N
    ("bhws,rs->bhwr", [[128, 14, 14, 256], [57, 256]]),   # K-major A, skinny N
    ("bshw,rs->brhw", [[128, 256, 14, 14], [57, 256]]),
    ("bshw,rs->bhwr", [[128, 256, 14, 14], [229, 256]]),
]
cases = eval(os.environ["CASES"]) if "CASES" in os.environ else DEFAULT
ctx = Context(0, "auto")
torch.cuda.set_stream(ctx.torch_stream)
tag = os.environ.get("TAG", "dbg=" + os.environ.get("CE_TC_DBG", "0"))
for expr, dims in cases:
    plan = ce.optimal(expr, dims, "same", "training")
    ex = Executor(ctx, plan)
    xs = [ctx.fill_random(d, 7 + i) for i, d in enumerate(dims)]
    for _ in range(3):
        ex.execute(xs)
    ex.set_profiling(True)
    best = {}
    for _ in range(5):
        ex.execute(xs)
        for n, k, t, fl, by in ex.profile(False):
            best[n] = min(best.get(n, 1e9), t)
            best[n + "#"] = (k, fl, by)
    ex.set_profiling(False)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(50):
        ex.execute(xs)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"{tag:8s} {expr:24s} loop {ev[0].elapsed_time(ev[1]) / 50 * 1e3:8.1f} us/execute")
    for n in [k for k in best if not k.endswith("#")]:
        k, fl, by = best[n + "#"]
        t = best[n]
        print(f"{tag:8s} {expr:24s} {str(dims):34s} {n:12s} {k:8s} {t*1e3:8.1f} us {fl/(t*1e-3)/1e12:7.1f} TF "
              f"{by/(t*1e-3)/1e9:7.0f} GB/s", flush=True)
    print(plan.describe_steps(False).strip().replace("\n", " ; "))
