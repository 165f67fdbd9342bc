import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_2401_03384_b200 as ce
from paper_2401_03384_b200.device import Context, Executor
import bench
res = {}
for mode in ["exec_graphs", "step_graph"]:
    ctx = Context(0, "auto", graphs=(mode == "exec_graphs"))
    st = ctx.torch_stream
    torch.cuda.set_stream(st)
    layers = []
    for kind, cr in bench.LAYERS:
        le = bench.layer_expr(kind, cr, 128)
        plan = ce.optimal(le.expr, le.dims, "same", "training")
        ex = Executor(ctx, plan, backward=True)
        xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
        dout = ctx.fill_random(plan.out_dims, 2000)
        layers.append((ex, xs, dout, torch.empty(plan.out_dims, device="cuda")))
    def step():
        for ex, xs, dout, out in layers:
            ex.execute(xs, out)
            ex.backward(xs, dout)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    run = step
    if mode == "step_graph":
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            step()
        torch.cuda.synchronize()
        run = g.replay
        for _ in range(3):
            run()
        torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    ts = []
    for _ in range(20):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[mode] = (statistics.mean(ts), min(ts))
    print(mode, res[mode], flush=True)
