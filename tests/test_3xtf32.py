"""3xTF32 math mode (CE_MATH_3XTF32; SURVEY §5's precision options): every tensor-core step
runs as hi*hi + hi*lo + lo*hi with hi = TF32(x) (round to nearest) and lo = x - hi, which keeps
the tensor cores and restores FP32-level accuracy.  Checked against the FP64 oracle at the
FP32 tolerance class (2e-5 normwise) where the TF32 context needs 5e-3 / 1e-2."""
import json

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from oracle import np_oracle as npo

LAYERS = [("cp", [32], [16], 3, 14, 4, [13]), ("tk", [32], [16], 3, 10, 4, [9, 7]),
          ("tt", [24], [16], 3, 9, 3, [5, 6, 7]), ("tr", [16], [16], 3, 8, 2, [3, 4, 5, 6]),
          ("standard", [16], [8], 3, 10, 2, [])]
TOL = 2e-5


def test_3xtf32_steps():
    kind, tf, sf, k, hp, b, r = LAYERS[1]
    le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, b, r))
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    steps = plan.describe_steps(True, "3xtf32").splitlines()
    tc = [s for s in steps if " tc " in s]
    assert tc and len([s for s in tc if "3xtf32-hl" in s]) * 3 == len(tc)
    assert sum(" split " in s for s in steps) == 2 * len(tc) // 3


@pytest.mark.gpu
@pytest.mark.parametrize("layer", LAYERS, ids=[l[0] for l in LAYERS])
def test_3xtf32_layer_vs_oracle(layer):
    import torch
    from paper_2401_03384_b200.device import Context, Executor
    c = Context(0, "3xtf32")
    kind, tf, sf, k, hp, b, r = layer
    le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, b, r))
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    ex = Executor(c, plan, backward=True)
    xs = [c.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    out = ex.execute(xs)
    dout = c.fill_random(plan.out_dims, 2000)
    grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    assert ex.stats.tc_steps > 0
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref_y, _ = npo.execute(le.expr, le.dims, nodes, ins)
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout.double().cpu().numpy())

    def nerr(y, ref):
        return float(np.abs(np.asarray(y, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))

    assert nerr(out.cpu().numpy(), ref_y) <= TOL
    for g, rr in zip(grads, ref_g):
        assert nerr(g.cpu().numpy(), rr) <= TOL


@pytest.mark.gpu
def test_3xtf32_full_size_tk():
    """cfg2 TK cr 1.0 (B=128): per-sample forward at FP32 accuracy on the tensor cores."""
    import torch
    from paper_2401_03384_b200.device import Context, Executor
    c = Context(0, "3xtf32")
    le = ce.expression(ce.LayerSpec("tk", [256], [256], 3, 3, 14, 14, 128, [1, 1]), 1.0)
    plan = ce.optimal(le.expr, le.dims, "same", "inference")
    ex = Executor(c, plan)
    xs = [c.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    out = ex.execute(xs)
    torch.cuda.synchronize()
    one = ce.expression(ce.LayerSpec("tk", [256], [256], 3, 3, 14, 14, 1, le.ranks))
    p1 = ce.optimal(one.expr, one.dims, "same", "inference")
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(p1.to_json())["nodes"]]
    ins = [xs[0][5:6].double().cpu().numpy()] + [x.double().cpu().numpy() for x in xs[1:]]
    ref, _ = npo.execute(one.expr, one.dims, nodes, ins)
    y = out[5:6].double().cpu().numpy()
    assert float(np.abs(y - ref).max() / np.abs(ref).max()) <= TOL
