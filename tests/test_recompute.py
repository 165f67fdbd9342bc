"""Gradient checkpointing: executors created with
recompute=True keep no forward intermediates; backward() recomputes them, so it needs no
preceding execute(), and every such executor of a context runs on one shared arena."""
import ctypes
import json

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from oracle import np_oracle as npo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_G = 1e-2


def _nerr(y, r):
    y = np.asarray(y, np.float64).ravel()
    r = np.asarray(r, np.float64).ravel()
    return float(np.abs(y - r).max() / max(np.abs(r).max(), 1e-30))


LAYERS = [("cp", [32], [16], 3, 14, 4, [13]), ("tk", [32], [16], 3, 10, 4, [9, 7]),
          ("tt", [24], [16], 3, 9, 3, [5, 6, 7]), ("rtr", [2, 2, 4], [2, 2, 2], 3, 8, 2, [3, 3, 3, 3])]


@pytest.mark.parametrize("layer", LAYERS, ids=[l[0] for l in LAYERS])
def test_recompute_matches_keep_and_oracle(ctx, layer):
    from paper_2401_03384_b200.device import Executor
    kind, tf, sf, k, hp, b, ranks = layer
    le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, b, ranks))
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    dout = ctx.fill_random(plan.out_dims, 2000)
    keep = Executor(ctx, plan, backward=True)
    keep.execute(xs)
    g_keep = keep.backward(xs, dout)
    rec = Executor(ctx, plan, backward=True, recompute=True)
    g_rec = rec.backward(xs, dout)  # no execute() first: the intermediates are recomputed
    out_rec = rec.execute(xs)
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref_y, _ = npo.execute(le.expr, le.dims, nodes, ins)
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout.double().cpu().numpy())
    assert _nerr(out_rec.cpu().numpy(), ref_y) <= 5e-3
    for a, b_, r in zip(g_keep, g_rec, ref_g):
        assert _nerr(b_.cpu().numpy(), r) <= TOL_G
        assert _nerr(b_.cpu().numpy(), a.cpu().numpy()) <= 1e-5  # same kernels, same order


def test_recompute_executors_share_one_arena():
    from paper_2401_03384_b200 import _lib
    from paper_2401_03384_b200.device import Context, Executor
    c = Context(0, "auto")
    exs, sizes = [], []
    for kind, tf, sf, k, hp, b, ranks in LAYERS:
        le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, b, ranks))
        plan = ce.optimal(le.expr, le.dims, "same", "training")
        ex = Executor(c, plan, backward=True, recompute=True)
        xs = [c.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
        ex.execute(xs)
        ex.backward(xs, c.fill_random(plan.out_dims, 2000))
        exs.append(ex)
        d = plan.describe_steps(True, "auto", recompute=True).splitlines()
        sizes.append(int([l for l in d if l.startswith("workspace_bytes ")][0].split()[1]))
    torch.cuda.synchronize()
    got = ctypes.c_size_t()
    _lib.check(_lib.lib().ce_ctx_workspace_bytes(c.handle, ctypes.byref(got)))
    assert got.value == max(sizes)
