"""Phase + per-iteration stamps of ONE TC launch inside a cfg2 layer's fwd+bwd (graphs off).
usage: CE_TC_DBG=544 CE_TC_DBG_AT=<n-th TC launch> python tools/tc_phases_layer.py tk 1.0 [T-factors S-factors K HP B]
       (default shape: the cfg2 layer 256 256 3 14 128; e.g. rtr 0.1 4,4,8 4,4,4 3 28 256)
Needs the debug build of the TC kernel (flags and stamps are compiled out otherwise):
  rm -rf build && make -C paper_2401_03384_b200/csrc TC_DEBUG=1   (rebuild normally afterwards)
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_03384_b200 as ce  # noqa: E402
from paper_2401_03384_b200 import _lib  # noqa: E402
from paper_2401_03384_b200.device import Context, Executor  # noqa: E402

kind, cr = sys.argv[1], float(sys.argv[2])
SL = {"cp": 1, "tk": 2, "tt": 3, "tr": 4, "rtr": 4, "rcp": 1, "rtk": 2, "rtt": 3}
ctx = Context(0, "auto", graphs=False)
torch.cuda.set_stream(ctx.torch_stream)
slots = SL[kind]
if len(sys.argv) > 7:
    tf, sf = ([int(x) for x in a.split(",")] for a in sys.argv[3:5])
    k, hp, B = (int(x) for x in sys.argv[5:8])
else:
    tf, sf, k, hp, B = [256], [256], 3, 14, 128
le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, B, [1] * slots), cr)
plan = ce.optimal(le.expr, le.dims, "same", "training")
ex = Executor(ctx, plan, backward=True)
xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
dout = ctx.fill_random(plan.out_dims, 2000)
ex.execute(xs)
ex.backward(xs, dout)
torch.cuda.synchronize()
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
it = (ctypes.c_ulonglong * 768)()
_lib.lib().ce_debug_tc_iter_timestamps(it)
a = np.array(it, dtype=np.float64).reshape(3, 256)
if (a > 0).any():
    base = a[a > 0].min()
    for role, nm in enumerate(["producer", "mma"]):
        v = a[role]
        v = (v[v > 0] - base) / 1.9e3
        print(nm, " ".join(f"{x:.2f}" for x in v[:60]))
    e = a[2].reshape(64, 4)
    e = e[e[:, 0] > 0]
    if len(e):
        e = (e - base) / 1.9e3
        print("epi [start, tables, tfull, stored] per tile:")
        for row in e[:int(os.environ.get("EPI_ROWS", "16"))]:
            print("   ", " ".join(f"{x:8.2f}" for x in row))
