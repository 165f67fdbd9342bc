"""GPU parity: every path through libce (C-ABI) against the FP64 oracle.

Tolerances (normwise max |y - y*| / max |y*|, SURVEY §8(c) C4 calibration):
  FP32 SIMT ("fp32" context)                 forward 1e-5,  gradients 1e-5
  auto (TF32 tensor cores where mapped)      forward 5e-3,  gradients 1e-2
Inputs are SplitMix64 (fill_random) rounded to FP32; the oracle is fed the same
rounded values in FP64.
"""
import json
import os

import numpy as np
import pytest

from oracle import np_oracle as npo
from tests.spec_gen import random_spec

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"fp32": (1e-5, 1e-5), "auto": (5e-3, 1e-2)}


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def nerr(y, ref):
    y = np.asarray(y, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    scale = max(np.abs(ref).max(), 1e-30)
    return float(np.abs(y - ref).max() / scale)


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def dev(x):
    return torch.tensor(np.asarray(x, dtype=np.float32), device="cuda:0").contiguous()


@pytest.fixture(params=["fp32", "auto"])
def any_ctx(request, ctx, ctx_simt):
    return (ctx_simt if request.param == "fp32" else ctx), request.param


def test_fill_random_device(ctx):
    t = ctx.fill_random([37, 41], 1234)
    ref = npo.fill_random([37, 41], 1234).astype(np.float32)
    assert np.array_equal(t.cpu().numpy(), ref)


def test_pairwise_golden(any_ctx):
    from paper_2401_03384_b200.device import pairwise_eval
    c_, mode = any_ctx
    tol = TOL[mode][0]
    for c in load("pairwise.json"):
        if "seeds" in c:
            a = npo.fill_random(c["ldims"], c["seeds"][0])
            b = npo.fill_random(c["rdims"], c["seeds"][1])
            op = npo.pairwise_from_expr(c["expr"], c["ldims"], c["rdims"], c["mode"])
            ref = npo.pairwise_eval(op, f32(a), f32(b))
        else:
            a, b = np.array(c["a"], float), np.array(c["b"], float)
            ref = np.array(c["out"]).reshape(c["rdims_out"])
        out = pairwise_eval(c_, c["expr"], dev(a).reshape(c["ldims"]), dev(b).reshape(c["rdims"]), c["mode"])
        torch.cuda.synchronize()
        assert list(out.shape) == list(c["rdims_out"])
        assert nerr(out.cpu().numpy(), ref) <= tol, (c["expr"], c["mode"])


def test_pairwise_grad_random(any_ctx):
    from paper_2401_03384_b200.device import pairwise_grad
    c_, mode = any_ctx
    tol = TOL[mode][1]
    rng = np.random.default_rng(11)
    n = 0
    while n < 120:
        expr, dims, cmode = random_spec(rng, 2, 2, dmax=6)
        try:
            op = npo.pairwise_from_expr(expr, dims[0], dims[1], cmode)
        except AssertionError:
            continue
        if any(ax.mode == "valid" and ax.feature < ax.filter for ax in op.conv):
            continue
        a = f32(rng.uniform(-1, 1, dims[0]))
        b = f32(rng.uniform(-1, 1, dims[1]))
        dc = f32(rng.uniform(-1, 1, op.result_dims))
        da_ref, db_ref = npo.pairwise_grad(op, a, b, dc)
        da, db = pairwise_grad(c_, expr, dev(a).reshape(dims[0]), dev(b).reshape(dims[1]),
                               dev(dc).reshape(op.result_dims), cmode)
        torch.cuda.synchronize()
        assert nerr(da.cpu().numpy(), da_ref) <= tol, (expr, cmode, "dA")
        assert nerr(db.cpu().numpy(), db_ref) <= tol, (expr, cmode, "dB")
        n += 1


def _run_plan(c_, expr, dims, mode, ins, dout=None, cost_mode="inference"):
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Executor
    plan = ce.optimal(expr, dims, mode, cost_mode)
    ex = Executor(c_, plan, backward=dout is not None)
    xs = [dev(x).reshape(d) for x, d in zip(ins, dims)]
    out = ex.execute(xs)
    grads = ex.backward(xs, dev(dout).reshape(plan.out_dims)) if dout is not None else None
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    return plan, nodes, out.cpu().numpy(), grads, ex


def test_execute_golden(any_ctx):
    c_, mode = any_ctx
    for c in load("execute.json"):
        ins = [f32(npo.fill_random(d, s)) for d, s in zip(c["dims"], c["seeds"])]
        plan, nodes, out, _, _ = _run_plan(c_, c["expr"], c["dims"], c["mode"], ins)
        ref, _ = npo.execute(c["expr"], c["dims"], nodes, ins, c["mode"])
        assert list(out.shape) == c["shape"]
        assert nerr(out, ref) <= TOL[mode][0], c["expr"]


def test_backward_random_specs(any_ctx):
    c_, mode = any_ctx
    rng = np.random.default_rng(21)
    n = 0
    while n < 60:
        expr, dims, cmode = random_spec(rng, 1, 5, dmax=4)
        import paper_2401_03384_b200 as ce
        try:
            plan = ce.optimal(expr, dims, cmode)
        except ce.CeError:
            continue
        ins = [f32(rng.uniform(-1, 1, d)) for d in dims]
        dout = f32(rng.uniform(-1, 1, plan.out_dims))
        plan, nodes, out, grads, _ = _run_plan(c_, expr, dims, cmode, ins, dout)
        ref_out, _ = npo.execute(expr, dims, nodes, ins, cmode)
        ref_g = npo.backward(expr, dims, nodes, ins, dout, cmode)
        assert nerr(out, ref_out) <= TOL[mode][0], expr
        for i, (g, r) in enumerate(zip(grads, ref_g)):
            assert nerr(g.cpu().numpy(), r) <= TOL[mode][1], (expr, i)
        n += 1


LAYER_CASES = [
    # (name, kind, T, S, Hp, B, cr or ranks)
    ("cfg1 CP", "cp", 64, 64, 32, 8, [16]),
    ("cfg2 TK cr0.1", "tk", 256, 256, 14, 128, 0.1),
    ("cfg2 TT cr0.1", "tt", 256, 256, 14, 128, 0.1),
    ("cfg2 TK cr1.0", "tk", 256, 256, 14, 128, 1.0),
    ("cfg2 TT cr1.0", "tt", 256, 256, 14, 128, 1.0),
    # cfg5 compression-sweep end points and the dense baseline at the cfg2 shape
    ("cfg5 CP cr0.5", "cp", 256, 256, 14, 128, 0.5),
    ("cfg5 TR cr0.05", "tr", 256, 256, 14, 128, 0.05),
    ("cfg5 TT cr0.05", "tt", 256, 256, 14, 128, 0.05),
    ("cfg5 dense", "standard", 256, 256, 14, 128, []),
    # cfg4 CP stack first layer (7x7 at 112x112, 3->64), reduced batch
    ("cfg4 CP conv1 cr1.0", "cp", 64, 3, 112, 8, 1.0),
    # R = 11: 3 lane quads, filter-gradient K slices capped (same-address atomics)
    ("cfg4 CP conv1 cr0.1 B32", "cp", 64, 3, 112, 32, 0.1),
]


def _layer(kind, T, S, Hp, B, cr):
    import paper_2401_03384_b200 as ce
    slots = {"cp": 1, "tk": 2, "tt": 3, "tr": 4, "standard": 0}[kind]
    k = 7 if (S == 3 and Hp == 112) else 3  # ResNet-34 conv1 is 7x7
    spec = ce.LayerSpec(kind, [T], [S], k, k, Hp, Hp, B, cr if isinstance(cr, list) else [1] * slots)
    return ce.expression(spec, None if isinstance(cr, list) else cr)


@pytest.mark.parametrize("case", LAYER_CASES, ids=[c[0] for c in LAYER_CASES])
def test_baseline_layers_full_size(any_ctx, case):
    """Full BASELINE shapes: per-sample forward vs the oracle (exact property: sample b depends only
    on X[b]) and gradients through the multilinear identity <dY,Y> = <dX,X> = <dW_i,W_i>."""
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Executor
    c_, mode = any_ctx
    name, kind, T, S, Hp, B, cr = case
    le = _layer(kind, T, S, Hp, B, cr)
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    ex = Executor(c_, plan, backward=True)
    xs = [c_.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    dout = c_.fill_random(plan.out_dims, 2000)
    out = ex.execute(xs)
    grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    # per-sample oracle check on two samples
    one = _layer(kind, T, S, Hp, 1, le.ranks if not isinstance(cr, list) else cr)
    p1 = ce.optimal(one.expr, one.dims, "same", "inference")
    nodes1 = [(n["left"], n["right"], n["result"]) for n in json.loads(p1.to_json())["nodes"]]
    for b in (0, B - 1):
        ins = [xs[0][b:b + 1].double().cpu().numpy()] + [x.double().cpu().numpy() for x in xs[1:]]
        ref, _ = npo.execute(one.expr, one.dims, nodes1, ins, "same")
        assert nerr(out[b:b + 1].cpu().numpy(), ref) <= TOL[mode][0], (name, b)
    y_dot = float((out.double() * dout.double()).sum())
    for i, (x, g) in enumerate(zip(xs, grads)):
        gx = float((g.double() * x.double()).sum())
        assert abs(gx - y_dot) <= TOL[mode][1] * max(abs(y_dot), 1e-6) * 10, (name, i, gx, y_dot)


def test_cp_layer_gradients_vs_oracle(any_ctx):
    """cfg1-shape CP layer at batch 2: every gradient against the FP64 adjoint oracle."""
    c_, mode = any_ctx
    le = _layer("cp", 64, 64, 32, 2, [16])
    rng = np.random.default_rng(4)
    ins = [f32(rng.uniform(-1, 1, d)) for d in le.dims]
    import paper_2401_03384_b200 as ce
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    dout = f32(rng.uniform(-1, 1, plan.out_dims))
    plan, nodes, out, grads, _ = _run_plan(c_, le.expr, le.dims, "same", ins, dout, "training")
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout)
    for g, r in zip(grads, ref_g):
        assert nerr(g.cpu().numpy(), r) <= TOL[mode][1]


def test_conv_einsum_autograd(ctx):
    """The paper's call form conv_einsum("...", T1, T2, ...) as a torch autograd op."""
    import paper_2401_03384_b200 as ce
    le = _layer("cp", 16, 12, 8, 3, [4])
    rng = np.random.default_rng(8)
    ins = [f32(rng.uniform(-1, 1, d)) for d in le.dims]
    xs = [dev(x).reshape(d).requires_grad_(True) for x, d in zip(ins, le.dims)]
    y = ce.conv_einsum(le.expr, *xs)
    dy = f32(rng.uniform(-1, 1, list(y.shape)))
    y.backward(dev(dy).reshape(y.shape))
    torch.cuda.synchronize()
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ref_y, _ = npo.execute(le.expr, le.dims, nodes, ins)
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dy)
    assert nerr(y.detach().cpu().numpy(), ref_y) <= TOL["auto"][0]
    for x, r in zip(xs, ref_g):
        assert nerr(x.grad.cpu().numpy(), r) <= TOL["auto"][1]


def test_graph_replay_and_pointer_change(ctx):
    """CUDA-graph replay must track new input pointers (re-capture) and stay correct."""
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Executor
    le = _layer("tk", 32, 24, 8, 4, [6, 5])
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    ex = Executor(ctx, plan, backward=True)
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    for seed in (1, 2, 2, 3):
        xs = [ctx.fill_random(d, seed * 100 + i) for i, d in enumerate(le.dims)]
        y = ex.execute(xs)
        torch.cuda.synchronize()
        ref, _ = npo.execute(le.expr, le.dims, nodes, [x.double().cpu().numpy() for x in xs])
        assert nerr(y.cpu().numpy(), ref) <= TOL["auto"][0]


def test_layer_zoo_forward_backward(any_ctx):
    """All 13 layer kinds (SPEC.md:569 toy dims) forward + every gradient vs the FP64 oracle."""
    import paper_2401_03384_b200 as ce
    c_, mode = any_ctx
    for case in load("layers.json")["layers"]:
        if case["cr"] > 0 or "cfg" in case["name"] or "dense" in case["name"]:
            continue
        rng = np.random.default_rng(17)
        ins = [f32(rng.uniform(-1, 1, d)) for d in case["dims"]]
        plan = ce.optimal(case["expr"], case["dims"], "same", "training")
        dout = f32(rng.uniform(-1, 1, plan.out_dims))
        plan, nodes, out, grads, _ = _run_plan(c_, case["expr"], case["dims"], "same", ins, dout, "training")
        ref, _ = npo.execute(case["expr"], case["dims"], nodes, ins)
        ref_g = npo.backward(case["expr"], case["dims"], nodes, ins, dout)
        assert nerr(out, ref) <= TOL[mode][0], case["name"]
        for i, (g, r) in enumerate(zip(grads, ref_g)):
            assert nerr(g.cpu().numpy(), r) <= TOL[mode][1], (case["name"], i)


@pytest.mark.parametrize("stage", ["conv1", "conv3_x", "conv5_x"])
def test_cp_resnet34_stage_shapes(ctx, stage):
    """cfg4 layer shapes (CP, cr=0.1) at batch 2: forward per sample + gradient identities."""
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Executor
    spec = dict(ce.resnet34_cp_blocks(2, 0.1))[stage]
    le = ce.expression(spec)
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    ex = Executor(ctx, plan, backward=True)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    dout = ctx.fill_random(plan.out_dims, 2000)
    out = ex.execute(xs)
    grads = ex.backward(xs, dout)
    torch.cuda.synchronize()
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ins = [x.double().cpu().numpy() for x in xs]
    ref, _ = npo.execute(le.expr, le.dims, nodes, ins)
    assert nerr(out.cpu().numpy(), ref) <= TOL["auto"][0]
    y_dot = float((out.double() * dout.double()).sum())
    for x, g in zip(xs, grads):
        gx = float((g.double() * x.double()).sum())
        assert abs(gx - y_dot) <= 1e-1 * max(abs(y_dot), 1e-6), (stage, gx, y_dot)


def test_rtr_cfg3_reduced(any_ctx):
    """cfg3 tensor-ring reshaped layer (64->64 as 4x4x4, M=3) at 14x14, batch 2: fwd + all grads."""
    import paper_2401_03384_b200 as ce
    c_, mode = any_ctx
    le = ce.expression(ce.LayerSpec("rtr", [4, 4, 4], [4, 4, 4], 3, 3, 14, 14, 2, [1, 1, 1, 1]), 0.1)
    rng = np.random.default_rng(23)
    ins = [f32(rng.uniform(-1, 1, d)) for d in le.dims]
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    dout = f32(rng.uniform(-1, 1, plan.out_dims))
    plan, nodes, out, grads, _ = _run_plan(c_, le.expr, le.dims, "same", ins, dout, "training")
    ref, _ = npo.execute(le.expr, le.dims, nodes, ins)
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout)
    assert nerr(out, ref) <= TOL[mode][0]
    for i, (g, r) in enumerate(zip(grads, ref_g)):
        assert nerr(g.cpu().numpy(), r) <= TOL[mode][1], i


def test_native_library_loaded(ctx):
    maps = open("/proc/self/maps").read()
    assert "libce.so" in maps


@pytest.mark.gpu
def test_flops_actual_and_conv_einsum_forward(ctx):
    """ce_flops_actual against the oracle; ce_conv_einsum (cached plan) against the FP64 oracle."""
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import conv_einsum_forward
    for e, d in [("bshw,rs->bhwr", [[8, 64, 32, 32], [16, 64]]), ("bhw(r2),(r1)(r2)hw->bhw(r1)|hw",
                                                                   [[2, 14, 14, 5], [6, 5, 3, 3]])]:
        assert ce.flops_actual(e, d) == npo.flops_actual(npo.pairwise_from_expr(e, d[0], d[1], "same"))
    expr, dims = "bshw,rt,rs,rh,rw->bthw|hw", [[2, 8, 9, 9], [4, 6], [4, 8], [4, 3], [4, 3]]
    rng = np.random.default_rng(5)
    ins = [f32(rng.uniform(-1, 1, d)) for d in dims]
    xs = [torch.from_numpy(x.astype(np.float32)).cuda() for x in ins]
    for _ in range(2):  # second call replays the cached executor
        out = conv_einsum_forward(ctx, expr, *xs)
    torch.cuda.synchronize()
    plan = ce.optimal(expr, dims, "same", "inference")
    nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(plan.to_json())["nodes"]]
    ref, _ = npo.execute(expr, dims, nodes, ins)
    assert nerr(out.cpu().numpy(), ref) <= TOL["auto"][0]


@pytest.mark.gpu
def test_single_rank_nccl_allreduce(ctx):
    """ce_nccl_unique_id / ce_ctx_init_comm / ce_allreduce_grads / ce_comm_wait on a 1-rank
    communicator: the SUM over one rank is the identity, and the comm stream is ordered
    after the context stream."""
    from paper_2401_03384_b200.device import Context, nccl_unique_id
    c = Context(0, "auto")
    c.init_comm(1, 0, nccl_unique_id())
    g = [torch.arange(1000, dtype=torch.float32, device="cuda"), torch.ones(7, device="cuda")]
    ref = [t.clone() for t in g]
    c.allreduce_grads(g)
    c.comm_wait()
    torch.cuda.synchronize()
    for a, b in zip(g, ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("conv_mode", ["same", "full", "valid"])
@pytest.mark.parametrize("rank", [20, 24, 18])
def test_depthwise_stencil_paths(any_ctx, conv_mode, rank):
    """Depthwise convolutions in every linear mode: the register-window stencil (forward and
    input gradient, all tap/position sign combinations) and the filter-gradient window kernel
    when the channel pitch is a multiple of 4 (rank 20, 24), the scalar stream path otherwise
    (18); every output and gradient against the FP64 oracle."""
    c_, mode = any_ctx
    rng = np.random.default_rng(31 + rank)
    for expr, dims in [("bhwr,rh->bhwr|h", [[6, 13, 9, rank], [rank, 3]]),
                       ("bhwr,rw->bhwr|w", [[5, 7, 11, rank], [rank, 5]]),
                       ("bhwr,rh->bhwr|h", [[4, 16, 3, rank], [rank, 7]])]:
        ins = [f32(rng.uniform(-1, 1, d)) for d in dims]
        import paper_2401_03384_b200 as ce
        plan = ce.optimal(expr, dims, conv_mode, "training")
        dout = f32(rng.uniform(-1, 1, plan.out_dims))
        plan, nodes, out, grads, _ = _run_plan(c_, expr, dims, conv_mode, ins, dout, "training")
        ref, _ = npo.execute(expr, dims, nodes, ins, conv_mode)
        ref_g = npo.backward(expr, dims, nodes, ins, dout, conv_mode)
        assert nerr(out, ref) <= TOL[mode][0], (expr, conv_mode, rank)
        for i, (g, r) in enumerate(zip(grads, ref_g)):
            assert nerr(g.cpu().numpy(), r) <= TOL[mode][1], (expr, conv_mode, rank, i)


PERMUTE_CASES = [
    # (expr, dims, expected kernel in describe)
    ("abcdef->dabcef", [4, 4, 4, 4, 28, 28], None),
    ("abcde->cbdae", [60, 60, 10, 10, 12], "block"),       # RTR pack: 4-wide unit axis out, 10-wide in
    ("abcde->abdce", [100, 120, 10, 16, 4], "block"),      # rowcopy with 10-wide rows
    ("ab->ba", [4, 1254400], "block"),                   # split axis: 1254400 = 448 x 2800
    ("abc->cab", [3, 4, 257], None),                     # prime extent: no block split, tile kernel
    ("abcd->dabc", [7, 9, 11, 13], None),
    ("bpqx->bxqp", [300, 784, 2, 10], "block"),          # RTR-like grad pack: 784 split 49 x 16
    ("ab->ba", [256, 1000], None),                       # 64x64 tile path
]


@pytest.mark.parametrize("case", PERMUTE_CASES, ids=[c[0] + "_" + "x".join(map(str, c[1])) for c in PERMUTE_CASES])
def test_permute_paths(ctx, case):
    """Unary permutes through every permute kernel, bit-exact against numpy (the block
    kernel is auto-selected from 4M elements on)."""
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Executor
    expr, dims, kind = case
    plan = ce.optimal(expr, [dims], "same", "inference")
    if kind:
        assert kind in plan.describe_steps(False), plan.describe_steps(False)
    x = ctx.fill_random(dims, 77)
    ex = Executor(ctx, plan)
    out = ex.execute([x])
    torch.cuda.synchronize()
    lhs, rhs = expr.split("->")
    ref = np.transpose(x.cpu().numpy(), [lhs.index(c) for c in rhs])
    assert np.array_equal(out.cpu().numpy(), ref)


RTR_X_FIRST = [  # (T factors, S factors, k, H, batch, tree): the path contracts X with the conv factor first
    ([4, 4, 8], [4, 4, 4], 3, 28, 1, "(((0 4) 1) (2 3))"),  # cfg3 64->128
    ([4, 4, 4], [1, 1, 3], 7, 56, 2, "(((0 4) 3) (1 2))"),  # cfg3 conv1 (7x7 taps), reduced
]


@pytest.mark.parametrize("case", RTR_X_FIRST, ids=["64to128_28", "conv1_56"])
def test_rtr_x_first_layers(any_ctx, case):
    """cfg3 RTR layers whose path starts with X * conv factor (tap expansion + TC, N=1 TC
    input gradient, block permutes of the 5-GB-class intermediates at full batch): fwd +
    all grads against the oracle at reduced batch."""
    import paper_2401_03384_b200 as ce
    c_, mode = any_ctx
    tf, sf, k, hp, batch, tree = case
    le = ce.expression(ce.LayerSpec("rtr", tf, sf, k, k, hp, hp, batch, [1, 1, 1, 1]), 0.1)
    rng = np.random.default_rng(29)
    ins = [f32(rng.uniform(-1, 1, d)) for d in le.dims]
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    assert plan.tree_encoding() == tree
    if mode == "auto":
        assert "expandA" in plan.describe_steps(True)
    dout = f32(rng.uniform(-1, 1, plan.out_dims))
    plan, nodes, out, grads, _ = _run_plan(c_, le.expr, le.dims, "same", ins, dout, "training")
    ref, _ = npo.execute(le.expr, le.dims, nodes, ins)
    ref_g = npo.backward(le.expr, le.dims, nodes, ins, dout)
    assert nerr(out, ref) <= TOL[mode][0]
    for i, (g, r) in enumerate(zip(grads, ref_g)):
        assert nerr(g.cpu().numpy(), r) <= TOL[mode][1], i


_PAIR_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2401_03384_b200 as ce
from paper_2401_03384_b200.device import Context, Executor
ctx = Context(0, "auto")
le = ce.expression(ce.LayerSpec("tk", [256], [256], 3, 3, 14, 14, 128, [1, 1]), 1.0)
plan = ce.optimal(le.expr, le.dims, "same", "training")
print(plan.describe_steps(True), file=sys.stderr)
ex = Executor(ctx, plan, backward=True)
xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
dout = ctx.fill_random(plan.out_dims, 2000)
out = ex.execute(xs)
grads = ex.backward(xs, dout)
torch.cuda.synchronize()
np.savez(sys.argv[2], out=out.cpu().numpy(), *[g.cpu().numpy() for g in grads])
"""


def test_cta_pair_path_opt_in(tmp_path):
    """CE_TC_PAIR=1 (cta_group::2 M=256 MMAs, B multicast, 2-CTA clusters) agrees with the
    default single-CTA path on the full cfg2 TK cr1.0 layer."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for flag in ("0", "1"):
        f = tmp_path / f"p{flag}.npz"
        env = dict(os.environ, CE_TC_PAIR=flag)
        r = subprocess.run([sys.executable, "-c", _PAIR_SCRIPT, root, str(f)], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        assert ("mc=2" in r.stderr) == (flag == "1"), r.stderr[-3000:]
        outs[flag] = np.load(f)
    for k in outs["0"].files:
        assert nerr(outs["1"][k], outs["0"][k]) <= 2e-3, k
