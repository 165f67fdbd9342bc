"""Per-kernel device times of one layer's fwd+bwd (profiling hooks).
usage: python tools/prof_layer.py KIND "T-factors" "S-factors" K HP B CR   e.g. cp "256" "256" 3 14 128 0.5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_03384_b200 as ce  # noqa: E402
from paper_2401_03384_b200.device import Context, Executor  # noqa: E402

kind, tf, sf, k, hp, b, cr = sys.argv[1:8]
tf = [int(x) for x in tf.split(",")]
sf = [int(x) for x in sf.split(",")]
slots = {"cp": 1, "tk": 2, "tt": 3, "tr": 4, "rtr": 4, "rcp": 1, "rtk": 2, "rtt": 3}[kind]
le = ce.expression(ce.LayerSpec(kind, tf, sf, int(k), int(k), int(hp), int(hp), int(b), [1] * slots), float(cr))
plan = ce.optimal(le.expr, le.dims, "same", "training")
print(le.expr, le.dims, le.ranks, plan.tree_encoding())
print(plan.describe_steps(True))
ctx = Context(0, "auto")
torch.cuda.set_stream(ctx.torch_stream)
ex = Executor(ctx, plan, backward=True)
xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
dout = ctx.fill_random(plan.out_dims, 2000)
for _ in range(2):
    ex.execute(xs)
    ex.backward(xs, dout)
ex.set_profiling(True)
ex.execute(xs)
f = ex.profile(False)
ex.backward(xs, dout)
bw = ex.profile(True)
torch.cuda.synchronize()
for n, kd, t, fl, by in f + bw:
    print(f"{n:22s} {kd:8s} {t*1e3:10.1f} us {fl/(t*1e-3)/1e12:7.2f} TF {by/(t*1e-3)/1e9:7.0f} GB/s")
print(f"total {sum(r[2] for r in f + bw)*1e3:10.1f} us")
