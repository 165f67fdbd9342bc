import torch, statistics, sys
sys.path.insert(0, ".")
import paper_2401_03384_b200 as ce
from paper_2401_03384_b200.device import Context, Executor
ctx = Context(0, "auto")
stream = ctx.torch_stream
torch.cuda.set_stream(stream)
layers = []
for kind, cr in [("tk", 0.1), ("tk", 1.0), ("tt", 0.1), ("tt", 1.0)]:
    le = ce.expression(ce.LayerSpec(kind, [256], [256], 3, 3, 14, 14, 128, [1] * {"tk": 2, "tt": 3}[kind]), cr)
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    ex = Executor(ctx, plan, backward=True)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    dout = ctx.fill_random(plan.out_dims, 2000)
    out = torch.empty(plan.out_dims, device="cuda")
    layers.append((ex, xs, dout, out))
def step():
    for ex, xs, dout, out in layers:
        ex.execute(xs, out)
        ex.backward(xs, dout)
for _ in range(3): step()
torch.cuda.synchronize()
flush = torch.empty(64 * 1024 * 1024, device="cuda")
def timeit(fn, n=20):
    ts = []
    for _ in range(n):
        flush.fill_(1.0); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); fn(); e1.record(stream); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts), statistics.median(ts)
print("eager (executor graphs)", timeit(step))
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g, stream=stream):
        step()
    print("captured with executor graphs inside")
    print("step graph", timeit(g.replay))
except Exception as e:
    print("capture failed:", e)
