"""Strided convolution (an extension -- the reference has no stride, SPEC.md:258,
481): a conv atom's mode may carry an output stride, "same/2" (or per atom "h=same/2,w=same/2").
Output position n reads feature index s*n + (the stride-1 map's offset), so a strided output is
exactly the stride-1 output at positions s*n -- which pins the strided oracle to the compiled
reference's stride-1 pairwise_eval.  The device lowers the forward and the filter gradient as
gathers with coefficient s and the feature gradient over a zero-upsampled dC.
"""
import json

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from oracle import np_oracle as npo

CASES = [  # (expr, ldims, rdims): the conv atoms h (and w) shared by both operands
    ("bsh,tsh->bth|h", [2, 3, 11], [4, 3, 3]),
    ("bshw,tshw->bthw|hw", [2, 3, 9, 7], [4, 3, 3, 3]),
    ("bhwr,rh->bhwr|h", [2, 10, 6, 5], [5, 3]),
    ("xh,h->xh|h", [3, 12], [5]),
]
MODES = ["same", "full", "valid", "circular"]


@pytest.fixture(params=["fp32", "auto"])
def any_ctx2(request, ctx, ctx_simt):
    """(context, (forward, gradient) tolerance): FP32 SIMT 1e-5, TF32 5e-3 / 1e-2."""
    return (ctx_simt, (1e-5, 1e-5)) if request.param == "fp32" else (ctx, (5e-3, 1e-2))


def _subsample(y, result, convs, s):
    idx = tuple(slice(None, None, s) if a in convs else slice(None) for a in result)
    return y[idx]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("stride", [2, 3])
def test_strided_oracle_is_subsampled_reference(ref, case, mode, stride):
    expr, ld, rd = case
    a = npo.fill_random(ld, 11)
    b = npo.fill_random(rd, 12)
    _, _, _, y1 = ref.pairwise(expr, [ld, rd], a, b, mode)
    op = npo.pairwise_from_expr(expr, ld, rd, f"{mode}/{stride}")
    ys = npo.pairwise_eval(op, a, b)
    convs = [ax.atom for ax in op.conv]
    assert np.allclose(ys, _subsample(y1, op.result, convs, stride), rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", MODES)
def test_strided_planner_dims_and_flops(mode):
    le = ce.expression(ce.LayerSpec("cp", [16], [8], 3, 3, 9, 9, 2, [5]))
    p = ce.optimal(le.expr, le.dims, f"{mode}/2", "training")
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(p.to_json())["nodes"]]
    ops, _ = npo.plan_ops(le.expr, le.dims, nodes, f"{mode}/2")
    assert p.flops_actual == sum(npo.flops_actual(op) for _, _, op in ops)
    h = npo.conv_output_dim(f"{mode}/2", 9, 3)
    assert p.out_dims == [2, 16, h, h]
    # stride 1 spelled explicitly is the reference's mode, bit for bit
    assert ce.optimal(le.expr, le.dims, f"{mode}/1").to_json() == ce.optimal(le.expr, le.dims, mode).to_json()


def test_per_atom_strides():
    le = ce.expression(ce.LayerSpec("cp", [16], [8], 3, 3, 9, 9, 2, [5]))
    p = ce.optimal(le.expr, le.dims, "h=same/2,w=same", "inference")
    assert p.out_dims == [2, 16, 5, 9]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["same/2", "full/2", "valid/2", "circular/2", "same/3"])
def test_strided_layer_forward_backward(any_ctx2, mode):
    """CP layer with both spatial atoms strided: forward and every gradient (the feature
    gradients go through the upsampled dC) against the oracle."""
    import torch
    from paper_2401_03384_b200.device import Executor
    c_, tol = any_ctx2
    le = ce.expression(ce.LayerSpec("cp", [12], [8], 3, 3, 11, 11, 2, [7]))
    plan = ce.optimal(le.expr, le.dims, mode, "training")
    ex = Executor(c_, plan, backward=True)
    xs = [c_.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    out = ex.execute(xs)
    dout = c_.fill_random(plan.out_dims, 2000)
    grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref_y, _ = npo.execute(le.expr, le.dims, nodes, ins, mode)
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout.double().cpu().numpy(), mode)

    def nerr(y, r):
        return float(np.abs(np.asarray(y, np.float64) - r).max() / max(np.abs(r).max(), 1e-30))

    assert list(out.shape) == list(ref_y.shape)
    assert nerr(out.cpu().numpy(), ref_y) <= tol[0]
    for g, r in zip(grads, ref_g):
        assert nerr(g.cpu().numpy(), r) <= tol[1]


@pytest.mark.gpu
def test_strided_resnet_downsampling_layer(ctx):
    """A true ResNet-34 stage transition (conv3_1: 64 -> 128, 3x3, stride 2, 56 -> 28) as a
    CP layer, batch 4, forward + gradients vs the oracle."""
    import torch
    from paper_2401_03384_b200.device import Executor
    le = ce.expression(ce.LayerSpec("cp", [128], [64], 3, 3, 56, 56, 4, [1]), 0.1)
    plan = ce.optimal(le.expr, le.dims, "same/2", "training")
    assert plan.out_dims == [4, 128, 28, 28]
    ex = Executor(ctx, plan, backward=True)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    out = ex.execute(xs)
    dout = ctx.fill_random(plan.out_dims, 2000)
    grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref_y, _ = npo.execute(le.expr, le.dims, nodes, ins, "same/2")
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout.double().cpu().numpy(), "same/2")
    e = float(np.abs(out.double().cpu().numpy() - ref_y).max() / np.abs(ref_y).max())
    assert e <= 5e-3
    for g, r in zip(grads, ref_g):
        assert float(np.abs(g.double().cpu().numpy() - r).max() / np.abs(r).max()) <= 1e-2
