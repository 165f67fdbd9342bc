"""Per-kernel times of one layer's fwd+bwd (profiling hooks); used for TC kernel experiments."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_03384_b200 as ce  # noqa: E402
from paper_2401_03384_b200.device import Context, Executor  # noqa: E402

kind, cr = sys.argv[1], float(sys.argv[2])
ctx = Context(0, os.environ.get("MATH", "auto"))
torch.cuda.set_stream(ctx.torch_stream)
slots = {"tk": 2, "tt": 3, "cp": 1, "tr": 4}[kind]
le = ce.expression(ce.LayerSpec(kind, [256], [256], 3, 3, 14, 14, 128, [1] * slots), cr)
plan = ce.optimal(le.expr, le.dims, "same", "training")
ex = Executor(ctx, plan, backward=True)
xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
dout = ctx.fill_random(plan.out_dims, 2000)
for _ in range(3):
    ex.execute(xs)
    ex.backward(xs, dout)
ex.set_profiling(True)
ex.execute(xs)
f = ex.profile(False)
ex.backward(xs, dout)
b = ex.profile(True)
torch.cuda.synchronize()
tag = os.environ.get("TAG", "")
for n, k, t, fl, by in f + b:
    print(f"{tag:10s} {n:20s} {k:8s} {t*1e3:9.1f} us  {fl/(t*1e-3)/1e12:7.1f} TF {by/(t*1e-3)/1e9:7.0f} GB/s")
print(f"{tag:10s} total {sum(r[2] for r in f + b)*1e3:9.1f} us")
