"""TEST INFRASTRUCTURE ONLY — FP64 numpy restatement of the reference executor.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use it,
and only as the checker.  Pinned against the compiled reference
(oracle/_ref/libconvexpr_ref.so) by tests/test_oracle.py and against the
committed golden vectors in tests/golden/.

Follows /root/reference/proj/src:
  make_pairwise_op      kernels.cpp:56-142
  sum_unique_modes      kernels.cpp:144-187
  canonicalize_operand  kernels.cpp:402-421
  grouped_conv_core     kernels.cpp:320-399 (feature_index 298-315, same_offset 52)
  pairwise_eval         kernels.cpp:425-470
  flops_actual          kernels.cpp:472-505
  execute               sequencer.cpp:403-447
The adjoint (pairwise_grad) has no reference counterpart (the reference has no
backward); it is the exact transpose of the same gather/select
computation and is validated against the reference's forward through the
bilinear identity <dC, f(A,B)> = <dA, A> = <dB, B> in tests/test_oracle.py.
"""
from __future__ import annotations

import itertools
import re
from dataclasses import dataclass, field

import numpy as np

_TOK = re.compile(r"\(([A-Za-z0-9]+)\)|([A-Za-z])")


def atoms(s: str):
    return [m.group(1) or m.group(2) for m in _TOK.finditer(s)]


def parse(expr: str):
    """(inputs, output, conv_atoms in output order) — valid expressions only."""
    expr = expr.replace(" ", "")
    lhs, rhs = expr.split("->")
    out, _, convs = rhs.partition("|")
    ins = [atoms(x) for x in lhs.split(",")]
    o = atoms(out)
    cl = atoms(convs.replace(",", ""))
    return ins, o, [a for a in o if a in cl]


def split_mode(mode):
    """"same" -> ("same", 1); "same/2" -> ("same", 2): the strided extension (ConvModeSpec in
    csrc/host/ce_ir.hpp; outside the reference's semantics)."""
    kind, _, st = mode.partition("/")
    return kind, int(st) if st else 1


def conv_output_dim(mode, x, l):
    kind, s = split_mode(mode)
    return {"full": (x + l - 2) // s + 1, "same": -(-x // s), "valid": (x - l) // s + 1, "circular": -(-x // s)}[kind]


def resolve_modes(ins, convs, mode):
    return {a: ("circular" if sum(a in s for s in ins) >= 3 else mode) for a in convs}


@dataclass
class ConvAxis:
    atom: str
    mode: str
    feature_on_left: bool
    feature: int
    filter: int
    out: int
    stride: int = 1


@dataclass
class Op:
    left: list
    right: list
    result: list
    ldims: list
    rdims: list
    result_dims: list = field(default_factory=list)
    conv: list = field(default_factory=list)
    batch: list = field(default_factory=list)
    contract: list = field(default_factory=list)
    lfree: list = field(default_factory=list)
    rfree: list = field(default_factory=list)
    lself: list = field(default_factory=list)
    rself: list = field(default_factory=list)
    dim: dict = field(default_factory=dict)


def make_op(left, ldims, right, rdims, keep, modes, result=None) -> Op:
    op = Op(list(left), list(right), [], list(ldims), list(rdims))
    kept = {}
    for i, a in enumerate(left):
        if a in right:
            dl, dr = ldims[i], rdims[right.index(a)]
            if a in modes:
                kind, st = split_mode(modes[a])
                ax = ConvAxis(a, kind, dl >= dr, max(dl, dr), min(dl, dr),
                              conv_output_dim(modes[a], max(dl, dr), min(dl, dr)), st)
                op.conv.append(ax)
                kept[a] = ax.out
                continue
            assert dl == dr, f"mismatched dims for {a}"
            (op.batch if a in keep else op.contract).append(a)
            op.dim[a] = dl
            if a in keep:
                kept[a] = dl
        else:
            (op.lfree if a in keep else op.lself).append(a)
            op.dim[a] = ldims[i]
            if a in keep:
                kept[a] = ldims[i]
    for j, a in enumerate(right):
        if a not in left:
            (op.rfree if a in keep else op.rself).append(a)
            op.dim[a] = rdims[j]
            if a in keep:
                kept[a] = rdims[j]
    if result is None:
        result = [a for a in left if a in kept] + [a for a in right if a in kept and a not in left]
    op.result = list(result)
    op.result_dims = [kept[a] for a in op.result]
    return op


def same_offset(l):
    return (l - 1) // 2


def feature_index(ax: ConvAxis, n, k):
    """Vectorised feature_index (kernels.cpp:298-315): (x, valid); a strided axis reads s*n."""
    n = n * ax.stride
    if ax.mode == "full":
        x = n - k
    elif ax.mode == "same":
        x = n + same_offset(ax.filter) - k
    elif ax.mode == "valid":
        x = n + k
    else:
        x = np.mod(n - k, ax.feature)
        return x, np.ones_like(x, dtype=bool)
    return x, (x >= 0) & (x < ax.feature)


def _canon(t, subs, op: Op, is_left):
    """Permute to [batch | contract | free | conv] and merge to [G,S,F,conv...]."""
    free = op.lfree if is_left else op.rfree
    order = [subs.index(a) for a in op.batch + op.contract + free] + [subs.index(ax.atom) for ax in op.conv]
    t = np.transpose(t, order)
    G = int(np.prod([op.dim[a] for a in op.batch])) if op.batch else 1
    S = int(np.prod([op.dim[a] for a in op.contract])) if op.contract else 1
    F = int(np.prod([op.dim[a] for a in free])) if free else 1
    conv = [(ax.feature if ax.feature_on_left == is_left else ax.filter) for ax in op.conv]
    return t.reshape([G, S, F] + conv)


def _taps(op):
    return itertools.product(*[range(ax.filter) for ax in op.conv])


def _select(t, op, is_left, taps):
    """Per tap combo: gather the feature side to [G,S,F,N] (N = prod out) or pick the filter index."""
    masks = []
    for i, ax in enumerate(op.conv):
        axis = 3 + i
        if ax.feature_on_left == is_left:
            x, valid = feature_index(ax, np.arange(ax.out), taps[i])
            t = np.take(t, np.where(valid, x, 0), axis=axis)
            shape = [1] * t.ndim
            shape[axis] = ax.out
            t = t * valid.reshape(shape)
        else:
            t = np.take(t, [taps[i]], axis=axis)
            t = np.repeat(t, ax.out, axis=axis)
    G, S, F = t.shape[:3]
    return t.reshape(G, S, F, -1)


def _unselect(g, shape, op, is_left, taps):
    """Exact adjoint of _select: scatter-add [G,S,F,N] back into the canonical operand."""
    G, S, F = shape[:3]
    outs = [ax.out for ax in op.conv]
    g = g.reshape([G, S, F] + outs)
    res = np.zeros(shape)
    # build index arrays per conv axis: position in operand for each out position n
    idx = []
    wts = []
    for i, ax in enumerate(op.conv):
        n = np.arange(ax.out)
        if ax.feature_on_left == is_left:
            x, valid = feature_index(ax, n, taps[i])
            idx.append(np.where(valid, x, 0))
            wts.append(valid.astype(np.float64))
        else:
            idx.append(np.full(ax.out, taps[i]))
            wts.append(np.ones(ax.out))
    if not op.conv:
        return g.reshape(shape)
    grids = np.meshgrid(*idx, indexing="ij")
    wgrid = np.ones(outs)
    for i, w in enumerate(wts):
        sh = [1] * len(outs)
        sh[i] = outs[i]
        wgrid = wgrid * w.reshape(sh)
    gw = g * wgrid
    flat_pos = np.ravel_multi_index([gr.ravel() for gr in grids], shape[3:])
    res2 = res.reshape(G, S, F, -1)
    np.add.at(res2, (slice(None), slice(None), slice(None), flat_pos), gw.reshape(G, S, F, -1))
    return res2.reshape(shape)


def _self_sum(t, subs, selfs):
    keep_axes = [i for i, a in enumerate(subs) if a not in selfs]
    drop = tuple(i for i, a in enumerate(subs) if a in selfs)
    return (t.sum(axis=drop) if drop else t), [subs[i] for i in keep_axes]


def _core_shape(op):
    return [op.dim[a] for a in op.batch] + [op.dim[a] for a in op.lfree] + [op.dim[a] for a in op.rfree] + \
           [ax.out for ax in op.conv], op.batch + op.lfree + op.rfree + [ax.atom for ax in op.conv]


def pairwise_eval(op: Op, a, b):
    a = np.asarray(a, dtype=np.float64).reshape(op.ldims)
    b = np.asarray(b, dtype=np.float64).reshape(op.rdims)
    la, lsubs = _self_sum(a, op.left, op.lself)
    rb, rsubs = _self_sum(b, op.right, op.rself)
    L = _canon(la, lsubs, op, True)
    R = _canon(rb, rsubs, op, False)
    G, _, FL = L.shape[:3]
    FR = R.shape[2]
    N = int(np.prod([ax.out for ax in op.conv])) if op.conv else 1
    core = np.zeros((G, FL, FR, N))
    for taps in _taps(op):
        core += np.einsum("gsan,gsbn->gabn", _select(L, op, True, taps), _select(R, op, False, taps))
    shape, subs = _core_shape(op)
    core = core.reshape(shape)
    return np.transpose(core, [subs.index(x) for x in op.result]).copy()


def pairwise_grad(op: Op, a, b, dc):
    """(dA, dB) = gradients of <dc, pairwise_eval(op, a, b)>."""
    a = np.asarray(a, dtype=np.float64).reshape(op.ldims)
    b = np.asarray(b, dtype=np.float64).reshape(op.rdims)
    la, lsubs = _self_sum(a, op.left, op.lself)
    rb, rsubs = _self_sum(b, op.right, op.rself)
    L = _canon(la, lsubs, op, True)
    R = _canon(rb, rsubs, op, False)
    G, _, FL = L.shape[:3]
    FR = R.shape[2]
    shape, subs = _core_shape(op)
    dcore = np.transpose(np.asarray(dc, dtype=np.float64).reshape(op.result_dims),
                         [op.result.index(x) for x in subs]).reshape(G, FL, FR, -1)
    dL = np.zeros(L.shape)
    dR = np.zeros(R.shape)
    for taps in _taps(op):
        Ls = _select(L, op, True, taps)
        Rs = _select(R, op, False, taps)
        dL += _unselect(np.einsum("gabn,gsbn->gsan", dcore, Rs), L.shape, op, True, taps)
        dR += _unselect(np.einsum("gabn,gsan->gsbn", dcore, Ls), R.shape, op, False, taps)

    def uncanon(d, t_red, subs_red, full, full_subs, is_left):
        free = op.lfree if is_left else op.rfree
        order_atoms = op.batch + op.contract + free + [ax.atom for ax in op.conv]
        perm_shape = [t_red.shape[subs_red.index(x)] for x in order_atoms]
        d = d.reshape(perm_shape)
        d = np.transpose(d, [order_atoms.index(x) for x in subs_red])
        # broadcast over self-contracted atoms
        exp = d.reshape([t_red.shape[subs_red.index(x)] if x in subs_red else 1 for x in full_subs])
        return np.broadcast_to(exp, full.shape).copy()

    return uncanon(dL, la, lsubs, a, op.left, True), uncanon(dR, rb, rsubs, b, op.right, False)


def flops_actual(op: Op) -> int:
    f = 1
    for a in op.batch + op.contract + op.lfree + op.rfree:
        f *= op.dim[a]
    for ax in op.conv:
        if ax.stride > 1:  # (extension) in-range (n, k) pairs counted directly
            n_, k_ = np.meshgrid(np.arange(ax.out), np.arange(ax.filter), indexing="ij")
            f *= int(feature_index(ax, n_, k_)[1].sum())
        elif ax.mode in ("full", "circular"):
            f *= ax.feature * ax.filter
        elif ax.mode == "valid":
            f *= (ax.feature - ax.filter + 1) * ax.filter
        else:
            off = same_offset(ax.filter)
            f *= sum(max(0, min(ax.filter - 1, n + off) - max(0, n + off - ax.feature + 1) + 1) for n in range(ax.out))
    return f


def pairwise_from_expr(expr, ldims, rdims, mode="same"):
    """The op ref_pairwise/ce_pairwise_eval build: keep = result atoms, order = result."""
    ins, out, convs = parse(expr)
    return make_op(ins[0], ldims, ins[1], rdims, set(out), resolve_modes(ins, convs, mode), out)


def plan_ops(expr, dims, nodes, mode="same"):
    """Ops of a plan given its nodes [(left, right, result_subs_string)] (plan_to_json)."""
    ins, out, convs = parse(expr)
    modes = resolve_modes(ins, convs, mode)
    subs = [list(s) for s in ins]
    dd = [list(d) for d in dims]
    ops = []
    for l, r, res in nodes:
        res_atoms = atoms(res)
        op = make_op(subs[l], dd[l], subs[r], dd[r], set(res_atoms), modes, res_atoms)
        ops.append((l, r, op))
        subs.append(op.result)
        dd.append(op.result_dims)
    return ops, out


def execute(expr, dims, nodes, inputs, mode="same"):
    """execute() (sequencer.cpp:403-447) over an explicit node list; returns (output, intermediates)."""
    ops, out = plan_ops(expr, dims, nodes, mode)
    vals = [np.asarray(x, dtype=np.float64).reshape(d) for x, d in zip(inputs, dims)]
    if not ops:
        ins, out, _ = parse(expr)
        t, s = _self_sum(vals[0], ins[0], [a for a in ins[0] if a not in out])
        return np.transpose(t, [s.index(a) for a in out]).copy(), []
    for l, r, op in ops:
        vals.append(pairwise_eval(op, vals[l], vals[r]))
    root = ops[-1][2]
    return np.transpose(vals[-1], [root.result.index(a) for a in out]).copy(), vals


def backward(expr, dims, nodes, inputs, dout, mode="same"):
    """Gradients of <dout, execute(...)> w.r.t. every input (FP64 adjoint pass)."""
    ops, out = plan_ops(expr, dims, nodes, mode)
    _, vals = execute(expr, dims, nodes, inputs, mode)
    n = len(dims)
    grads = [None] * (n + len(ops))
    if not ops:
        ins, _, _ = parse(expr)
        d = np.asarray(dout, dtype=np.float64).reshape([dims[0][ins[0].index(a)] for a in out])
        exp = np.transpose(d, [out.index(a) for a in ins[0] if a in out])
        shape = [dims[0][i] if a in out else 1 for i, a in enumerate(ins[0])]
        return [np.broadcast_to(exp.reshape(shape), dims[0]).copy()]
    root = ops[-1][2]
    grads[-1] = np.transpose(np.asarray(dout, dtype=np.float64).reshape([root.result_dims[root.result.index(a)] for a in out]),
                             [out.index(a) for a in root.result])
    for j in reversed(range(len(ops))):
        l, r, op = ops[j]
        da, db = pairwise_grad(op, vals[l], vals[r], grads[n + j])
        grads[l], grads[r] = da, db
    return grads[:n]


def fill_random(shape, seed):
    """fill_random (tensor.cpp:107-130) vectorised: element i uses state seed+(i+1)*golden."""
    n = int(np.prod(shape)) if len(shape) else 1
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (np.arange(1, n + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (2.0 * u - 1.0).reshape(shape)
