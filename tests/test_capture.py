"""Executors inside a caller's CUDA-graph capture (a whole training step captured once and
replayed, as bench.py does at N=1): the steps launch straight into the caller's graph, and a
replay reproduces the eager results on new input values."""
import pytest

import paper_2401_03384_b200 as ce

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_step_graph_replay_matches_eager(ctx):
    from paper_2401_03384_b200.device import Executor
    stream = ctx.torch_stream
    torch.cuda.set_stream(stream)
    le = ce.expression(ce.LayerSpec("tk", [64], [32], 3, 3, 12, 12, 8, [1, 1]), 0.25)
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    ex = Executor(ctx, plan, backward=True)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    dout = ctx.fill_random(plan.out_dims, 2000)
    out = torch.empty(plan.out_dims, device="cuda")
    grads = [torch.empty_like(x) for x in xs]

    def step():
        ex.execute(xs, out)
        gs = ex.backward(xs, dout)
        for g, d in zip(grads, gs):
            g.copy_(d)

    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step()
    # new input values in the same buffers, then replay vs eager
    for i, x in enumerate(xs):
        x.copy_(ctx.fill_random(list(x.shape), 3000 + i))
    g.replay()
    torch.cuda.synchronize()
    y_graph, g_graph = out.clone(), [t.clone() for t in grads]
    step()
    torch.cuda.synchronize()
    assert torch.allclose(y_graph, out, rtol=0, atol=1e-5 * float(out.abs().max()))
    for a, b in zip(g_graph, grads):
        assert torch.allclose(a, b, rtol=0, atol=1e-5 * float(b.abs().max()))
