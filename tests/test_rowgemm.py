"""Row-GEMM kernel (csrc/cuda/ce_rowgemm.cu): rank contractions with K, N <= 32 over millions
of pixel rows (RTR conv1's node1 / node3 and their adjoints, CP conv1's 3-channel 1x1).  The
row threshold is lowered (CE_ROWGEMM_MIN) so small shapes take the kernel; forward and all
gradients against the FP64 oracle."""
import json

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from oracle import np_oracle as npo

CASES = [  # (kind, T factors, S factors, k, H, batch, cr)
    ("rtr", [4, 4, 4], [1, 1, 3], 7, 30, 2, 0.1),
    ("rtr", [2, 2, 2], [1, 1, 2], 3, 17, 3, 0.1),
    ("cp", [16], [3], 7, 20, 2, 0.1),
]


def _plan(case):
    kind, tf, sf, k, hp, b, cr = case
    slots = {"cp": 1, "rtr": 4}[kind]
    le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, b, [1] * slots), cr)
    return le, ce.optimal(le.expr, le.dims, "same", "training")


def test_rowgemm_routing(monkeypatch):
    monkeypatch.setenv("CE_ROWGEMM_MIN", "0")
    _, plan = _plan(CASES[0])
    assert " row rows=" in plan.describe_steps(True)
    monkeypatch.setenv("CE_ROWGEMM_MIN", str(1 << 40))
    assert " row rows=" not in plan.describe_steps(True)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=["rtr7", "rtr3", "cp7"])
def test_rowgemm_layer_vs_oracle(monkeypatch, ctx, case):
    import torch
    from paper_2401_03384_b200.device import Executor
    monkeypatch.setenv("CE_ROWGEMM_MIN", "0")
    le, plan = _plan(case)
    assert " row rows=" in plan.describe_steps(True)
    ex = Executor(ctx, plan, backward=True)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    out = ex.execute(xs)
    dout = ctx.fill_random(plan.out_dims, 2000)
    grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref_y, _ = npo.execute(le.expr, le.dims, nodes, ins)
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout.double().cpu().numpy())

    def nerr(y, r):
        return float(np.abs(np.asarray(y, np.float64) - r).max() / max(np.abs(r).max(), 1e-30))

    assert nerr(out.cpu().numpy(), ref_y) <= 5e-3
    for i, (g, r) in enumerate(zip(grads, ref_g)):
        assert nerr(g.cpu().numpy(), r) <= 1e-2, i
