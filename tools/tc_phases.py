"""Phase timestamps of one TC launch (CE_TC_DBG=32): python tools/tc_phases.py tk 0.1 <step-label>
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
from paper_2401_03384_b200.device import Context, pairwise_eval  # noqa: E402

ctx = Context(0, "auto", graphs=False)
torch.cuda.set_stream(ctx.torch_stream)
# the first GEMM of the TK layer: X (packed) . W2
expr = os.environ.get("EXPR", "bshw,rs->bhwr")
dims = eval(os.environ.get("DIMS", "[[128,256,14,14],[57,256]]"))
a = ctx.fill_random(dims[0], 1)
b = ctx.fill_random(dims[1], 2)
for _ in range(3):
    pairwise_eval(ctx, expr, a, b)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (160 * 16))()
_lib.lib().ce_debug_tc_timestamps(buf, 160 * 16)
ts = np.array(buf, dtype=np.float64).reshape(160, 16)[:148]
ts = ts[ts[:, 0] > 0]
t0 = ts[:, 0].min()
names = ["start", "setup", "producer_end", "mma_end", "epi_first_tile", "epi_end", "end", "first_stage", "prod_first_issue", "prod_enter", "epi_tables"]
for i, n in enumerate(names):
    v = (ts[:, i] - t0) / 1e3
    print(f"{n:16s} min {v.min():8.2f} us  median {np.median(v):8.2f} us  max {v.max():8.2f} us")
if int(os.environ["CE_TC_DBG"]) & 512:
    it = (ctypes.c_ulonglong * 768)()
    _lib.lib().ce_debug_tc_iter_timestamps(it)
    a = np.array(it, dtype=np.float64).reshape(3, 256)
    base = a[a > 0].min()
    for role, nm in enumerate(["producer", "mma", "commit"]):
        v = a[role]
        v = (v[v > 0] - base) / 1.9e3  # SM cycles -> us at ~1.9 GHz
        print(nm, " ".join(f"{x:.2f}" for x in v[:100]))
