"""Run one layer forward+backward a few times (for ncu captures).
usage: python tools/run_layer.py tk 1.0 [iters] [T S k Hp B]   (default: the cfg2 shape 256 256 3 14 128)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_03384_b200 as ce  # noqa: E402
from paper_2401_03384_b200.device import Context, Executor  # noqa: E402

kind, cr = sys.argv[1], float(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ctx = Context(0, "auto")
torch.cuda.set_stream(ctx.torch_stream)
slots = {"tk": 2, "tt": 3, "cp": 1, "tr": 4}[kind]
T, S, k, hp, B = (int(x) for x in sys.argv[4:9]) if len(sys.argv) > 8 else (256, 256, 3, 14, 128)
le = ce.expression(ce.LayerSpec(kind, [T], [S], k, k, hp, hp, B, [1] * slots), cr)
plan = ce.optimal(le.expr, le.dims, "same", "training")
print(plan.describe_steps(True), flush=True)
ex = Executor(ctx, plan, backward=True)
xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
dout = ctx.fill_random(plan.out_dims, 2000)
for _ in range(iters):
    ex.execute(xs)
    ex.backward(xs, dout)
torch.cuda.synchronize()
print("done")
