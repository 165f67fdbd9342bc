"""Phase + per-iteration timestamps of the factor-gradient (dB) TC launch of one pairwise node.
EXPR/DIMS env as in tc_phases.py; CE_TC_DBG = 32 | EXTRA_DBG.
Needs the debug build of the TC kernel (flags and stamps are compiled out otherwise):
  rm -rf build && make -C paper_2401_03384_b200/csrc TC_DEBUG=1   (rebuild normally afterwards)
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CE_TC_DBG"] = str(32 | int(os.environ.get("EXTRA_DBG", "0")))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_03384_b200 as ce  # noqa: E402
from paper_2401_03384_b200 import _lib  # noqa: E402
from paper_2401_03384_b200.device import Context, Executor  # noqa: E402

ctx = Context(0, "auto", graphs=False)
torch.cuda.set_stream(ctx.torch_stream)
expr = os.environ["EXPR"]
dims = eval(os.environ["DIMS"])
plan = ce.optimal(expr, dims, "same", "training")
print(plan.describe_steps(True))
ex = Executor(ctx, plan, backward=True)
xs = [ctx.fill_random(d, 1 + i) for i, d in enumerate(dims)]
dout = ctx.fill_random(plan.out_dims, 9)
needs = [os.environ.get("WHICH", "B") == "A", os.environ.get("WHICH", "B") == "B"]
for _ in range(3):
    ex.execute(xs)
    ex.backward(xs, dout, needs)
torch.cuda.synchronize()
ex.set_profiling(True)
ex.backward(xs, dout, needs)
torch.cuda.synchronize()
for n, k, t, fl, by in ex.profile(True):
    print(f"{n:20s} {k:8s} {t*1e3:9.1f} us  {fl/(t*1e-3)/1e12:7.1f} TF {by/(t*1e-3)/1e9:7.0f} GB/s")
buf = (ctypes.c_ulonglong * (160 * 16))()
_lib.lib().ce_debug_tc_timestamps(buf, 160 * 16)
ts = np.array(buf, dtype=np.float64).reshape(160, 16)[:148]
ts = ts[ts[:, 0] > 0]
t0 = ts[:, 0].min()
names = ["start", "setup", "producer_end", "mma_end", "epi_first_tile", "epi_end", "end", "first_stage", "prod_first_issue", "prod_enter", "epi_tables"]
for i, n in enumerate(names):
    v = (ts[:, i] - t0) / 1e3
    v = v[v >= 0]
    if len(v):
        print(f"{n:16s} min {v.min():8.2f} us  median {np.median(v):8.2f} us  max {v.max():8.2f} us")
if int(os.environ["CE_TC_DBG"]) & 512:
    it = (ctypes.c_ulonglong * 768)()
    _lib.lib().ce_debug_tc_iter_timestamps(it)
    a = np.array(it, dtype=np.float64).reshape(3, 256)
    base = a[a > 0].min()
    for role, nm in enumerate(["producer", "mma", "commit"]):
        v = a[role]
        v = (v[v > 0] - base) / 1.9e3
        print(nm, " ".join(f"{x:.2f}" for x in v[:100]))
