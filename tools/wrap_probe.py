import sys, torch
sys.path.insert(0, '.')
import paper_2401_03384_b200 as ce
from paper_2401_03384_b200.device import Context, Executor
math = sys.argv[1] if len(sys.argv) > 1 else "auto"
ctx = Context(0, math)
torch.cuda.set_stream(ctx.torch_stream)
le = ce.expression(ce.LayerSpec("cp", [32], [16], 3, 3, 14, 14, 4, [13]))
plan = ce.optimal(le.expr, le.dims, "same", "inference")
ex = Executor(ctx, plan)
xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
y = ex.execute(xs)
torch.cuda.synchronize()
print("ok", float(y.abs().sum()))
