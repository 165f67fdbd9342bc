"""Node fusion along plan chains: two chained depthwise stencils (the CP
layer's `bhwr,rh->bhwr` -> `bhwr,rw->bhwr`, layers.cpp:184-190, and their input-gradient
adjoints in the backward pass) run as one fused step (csrc/cuda/ce_fuse.cu).

Host-only tests check the step lists (the planner fuses exactly those pairs, stores the
intermediate only when a later step reads it); -m gpu tests check the fused executor against
the FP64 oracle, forward-only (intermediate never stored) and forward+backward, for every
tap count the kernel instantiates (3/5/7) and the Same/Full/Valid modes.
"""
import json

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from oracle import np_oracle as npo

TOL = (5e-3, 1e-2)  # TF32 context (the fused stencil itself is FP32; the 1x1 nodes run on TF32)


def _cp(S, T, k, hp, B, R):
    return ce.expression(ce.LayerSpec("cp", [T], [S], k, k, hp, hp, B, [R]))


def _steps(plan, backward):
    return [l for l in plan.describe_steps(backward, "auto").splitlines() if l.startswith(("fwd", "bwd"))]


def test_fused_steps_forward_only():
    le = _cp(64, 64, 3, 56, 8, 27)
    plan = ce.optimal(le.expr, le.dims, "same", "inference")
    steps = _steps(plan, False)
    fused = [s for s in steps if " dw2 " in s]
    assert len(fused) == 1 and "store_mid=0" in fused[0], steps


def test_fused_steps_training():
    le = _cp(64, 64, 3, 56, 8, 27)
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    steps = _steps(plan, True)
    fused = [s for s in steps if " dw2 " in s]
    # forward pair (its intermediate feeds the backward's filter gradient) + backward pair
    assert len(fused) == 2 and all("store_mid=1" in s for s in fused), steps
    assert not any(" dw2 " in l for l in plan.describe_steps(True, "fp32").splitlines())


def _run(ctx, le, mode, backward, cost="training"):
    import torch
    from paper_2401_03384_b200.device import Executor
    plan = ce.optimal(le.expr, le.dims, mode, cost)
    ex = Executor(ctx, plan, backward=backward)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    out = ex.execute(xs)
    grads = None
    dout = None
    if backward:
        dout = ctx.fill_random(plan.out_dims, 2000)
        grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref, _ = npo.execute(le.expr, le.dims, nodes, ins, mode)
    return plan, out, grads, dout, ins, nodes, ref


def _nerr(y, r):
    y = np.asarray(y, np.float64).ravel()
    r = np.asarray(r, np.float64).ravel()
    return float(np.abs(y - r).max() / max(np.abs(r).max(), 1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("k,hp,R", [(3, 14, 23), (5, 13, 11), (7, 15, 9), (3, 40, 37)])
@pytest.mark.parametrize("backward", [False, True])
def test_fused_cp_layer_matches_oracle(ctx, k, hp, R, backward):
    le = _cp(16, 24, k, hp, 4, R)
    plan, out, grads, dout, ins, nodes, ref = _run(ctx, le, "same", backward,
                                                   "training" if backward else "inference")
    assert any(" dw2 " in s for s in _steps(plan, backward))
    assert _nerr(out.cpu().numpy(), ref) <= TOL[0]
    if backward:
        ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout.double().cpu().numpy())
        for g, r in zip(grads, ref_g):
            assert _nerr(g.cpu().numpy(), r) <= TOL[1]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["full", "valid"])
def test_fused_stencil_modes(ctx, mode):
    """Full / Valid gathers (x = n - k / n + k and their adjoints) through the fused path,
    on the raw CP expression (not a layer) so the mode applies to both conv atoms."""
    import torch
    from paper_2401_03384_b200.device import Executor
    expr = "bshw,rt,rs,rh,rw->bthw|hw"
    dims = [[3, 16, 13, 11], [9, 20], [9, 16], [9, 3], [9, 3]]
    plan = ce.optimal(expr, dims, mode, "training")
    steps = _steps(plan, True)
    ex = Executor(ctx, plan, backward=True)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(dims)]
    out = ex.execute(xs)
    dout = ctx.fill_random(plan.out_dims, 2000)
    grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref, _ = npo.execute(expr, dims, nodes, ins, mode)
    ref_g = npo.backward(expr, dims, nodes, ins, dout.double().cpu().numpy(), mode)
    assert _nerr(out.cpu().numpy(), ref) <= TOL[0], steps
    for g, r in zip(grads, ref_g):
        assert _nerr(g.cpu().numpy(), r) <= TOL[1], steps
