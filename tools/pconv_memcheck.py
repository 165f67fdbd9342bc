import os, sys, torch
sys.path.insert(0, '.')
os.environ["CE_PCONV_MIN"] = "0"
import paper_2401_03384_b200 as ce
from paper_2401_03384_b200.device import Context, Executor
ctx = Context(0, "auto")
torch.cuda.set_stream(ctx.torch_stream)
for tf, sf, k, hp, b in [([4, 4, 4], [1, 1, 3], 7, 30, 2), ([2, 2, 2], [1, 1, 2], 5, 21, 3)]:
    for mode in ["same", "full", "valid"]:
        le = ce.expression(ce.LayerSpec("rtr", tf, sf, k, k, hp, hp, b, [1, 1, 1, 1]), 0.1)
        plan = ce.optimal(le.expr, le.dims, mode, "training")
        ex = Executor(ctx, plan, backward=True)
        xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
        y = ex.execute(xs)
        g = ex.backward(xs, ctx.fill_random(plan.out_dims, 2000))
        torch.cuda.synchronize()
print("ok")
