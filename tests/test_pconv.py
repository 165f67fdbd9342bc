"""Plane-conv kernels (csrc/cuda/ce_pconv.cu): convolutions whose feature operand is gathered
on two spatial axes against a small filter -- RTR conv1's X * W4 and its adjoints
(grouped_conv_core, kernels.cpp:320-399).  The position threshold is lowered
(CE_PCONV_MIN) so small shapes take the kernels; forward and every gradient are checked
against the FP64 oracle, in all four conv modes and with ragged tiles (positions not a
multiple of the 32 x 32 / 16 x 32 tiles)."""
import json

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from oracle import np_oracle as npo

CASES = [  # (T factors, S factors, k, H, batch)
    ([4, 4, 4], [1, 1, 3], 7, 30, 2),   # conv1-like: 7x7 taps, 9 output channels per plane
    ([2, 2, 2], [1, 1, 2], 5, 21, 3),   # 5x5 taps, ragged tiles
    ([2, 2, 2], [1, 2, 2], 3, 17, 2),   # 3x3 taps
]


def _plan(case, mode):
    tf, sf, k, hp, b = case
    le = ce.expression(ce.LayerSpec("rtr", tf, sf, k, k, hp, hp, b, [1, 1, 1, 1]), 0.1)
    return le, ce.optimal(le.expr, le.dims, mode, "training")


def test_pconv_routing(monkeypatch):
    monkeypatch.setenv("CE_PCONV_MIN", "0")
    le, plan = _plan(CASES[0], "same")
    steps = plan.describe_steps(True)
    assert "pconv kind=0" in steps and "pconv kind=1" in steps, steps
    monkeypatch.setenv("CE_PCONV_MIN", str(1 << 40))
    assert "pconv" not in plan.describe_steps(True)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=["7x7", "5x5", "3x3"])
@pytest.mark.parametrize("mode", ["same", "full", "valid"])
def test_pconv_layer_vs_oracle(monkeypatch, ctx, case, mode):
    import torch
    from paper_2401_03384_b200.device import Executor
    monkeypatch.setenv("CE_PCONV_MIN", "0")
    le, plan = _plan(case, mode)
    ex = Executor(ctx, plan, backward=True)
    steps = plan.describe_steps(True)
    assert "pconv" in steps, steps
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    out = ex.execute(xs)
    dout = ctx.fill_random(plan.out_dims, 2000)
    grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref_y, _ = npo.execute(le.expr, le.dims, nodes, ins, mode)
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout.double().cpu().numpy(), mode)

    def nerr(y, r):
        return float(np.abs(np.asarray(y, np.float64) - r).max() / max(np.abs(r).max(), 1e-30))

    assert nerr(out.cpu().numpy(), ref_y) <= 5e-3
    for i, (g, r) in enumerate(zip(grads, ref_g)):
        assert nerr(g.cpu().numpy(), r) <= 1e-2, i
