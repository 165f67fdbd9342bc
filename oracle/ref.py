"""TEST INFRASTRUCTURE ONLY — ctypes view of the compiled, unmodified reference.

`oracle/_ref/libconvexpr_ref.so` is built by `oracle/Makefile` from
/root/reference/proj/src/*.cpp plus our `ref_capi.cpp` shim.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may import
this module; the product path never does.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libconvexpr_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = ctypes.c_char_p
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _dims(dims):
    flat = [int(d) for ds in dims for d in ds]
    ranks = [len(ds) for ds in dims]
    return (ctypes.c_int64 * max(1, len(flat)))(*flat), (ctypes.c_int * len(ranks))(*ranks), len(ranks)


def _buf(n=1 << 20):
    return ctypes.create_string_buffer(n)


def plan(expr, dims, mode="same", cost_mode="inference", which="optimal", capped=False):
    """Returns (plan_json, tree_encoding, inference_cost, training_cost)."""
    d, r, n = _dims(dims)
    out = _buf()
    _check(lib().ref_plan(expr.encode(), d, r, n, mode.encode(), cost_mode.encode(),
                          0 if which == "optimal" else 1, int(capped), out, len(out)))
    js, enc, costs = out.value.decode().split("\n")
    ci, ct = costs.split()
    return js, enc, int(ci), int(ct)


def enumerate_min(expr, dims, mode="same", cost_mode="inference"):
    d, r, n = _dims(dims)
    out = _buf(256)
    _check(lib().ref_enumerate(expr.encode(), d, r, n, mode.encode(), cost_mode.encode(), out, len(out)))
    cnt, best = out.value.decode().split()
    return int(cnt), int(best)


def _inputs(arrs):
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in arrs]
    ptrs = (ctypes.POINTER(ctypes.c_double) * len(arrs))(
        *[a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for a in arrs])
    return arrs, ptrs


def execute(expr, dims, inputs, out_shape, mode="same", which="optimal"):
    """Reference execute(); returns (output ndarray, multiplications, peak, seconds)."""
    d, r, n = _dims(dims)
    keep, ptrs = _inputs(inputs)
    out = np.zeros(int(np.prod(out_shape)) if len(out_shape) else 1, dtype=np.float64)
    info = _buf(256)
    _check(lib().ref_execute(expr.encode(), d, r, n, mode.encode(), 0 if which == "optimal" else 1,
                             ptrs, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                             ctypes.c_int64(out.size), info, len(info)))
    m, p, s = info.value.decode().split()
    del keep
    return out.reshape(out_shape), int(m), int(p), float(s)


def time_execute(expr, dims, inputs, mode="same", cost_mode="inference", reps=3):
    d, r, n = _dims(dims)
    keep, ptrs = _inputs(inputs)
    best = ctypes.c_double()
    _check(lib().ref_time_execute(expr.encode(), d, r, n, mode.encode(), cost_mode.encode(), ptrs,
                                  int(reps), ctypes.byref(best)))
    del keep
    return best.value


def time_execute_mults(expr, dims, inputs, mode="same", cost_mode="inference", reps=1):
    """(best seconds, ExecutionResult.multiplications) of the reference execute()."""
    d, r, n = _dims(dims)
    keep, ptrs = _inputs(inputs)
    best = ctypes.c_double()
    out = _buf(128)
    _check(lib().ref_time_execute2(expr.encode(), d, r, n, mode.encode(), cost_mode.encode(), ptrs,
                                   int(reps), ctypes.byref(best), out, len(out)))
    del keep
    return best.value, int(out.value.decode())


def eval_brute(expr, dims, inputs, out_shape, mode="same"):
    d, r, n = _dims(dims)
    keep, ptrs = _inputs(inputs)
    out = np.zeros(max(1, int(np.prod(out_shape))), dtype=np.float64)
    _check(lib().ref_eval_brute(expr.encode(), d, r, n, mode.encode(), ptrs,
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_int64(out.size)))
    del keep
    return out.reshape(out_shape)


def pairwise(expr, dims, a=None, b=None, mode="same"):
    """Returns (flops_actual, (fwd, g1, g2) training costs, result_dims, result or None)."""
    d, r, _ = _dims(dims)
    info = _buf(1024)
    res = None
    if a is not None:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
    # first call with no data to learn the result shape
    _check(lib().ref_pairwise(expr.encode(), d, r, mode.encode(), None, None, None,
                              ctypes.c_int64(0), info, len(info)))
    parts = [int(x) for x in info.value.decode().split()]
    fa, costs, rdims = parts[0], tuple(parts[1:4]), parts[4:]
    if a is not None:
        res = np.zeros(max(1, int(np.prod(rdims))), dtype=np.float64)
        P = ctypes.POINTER(ctypes.c_double)
        _check(lib().ref_pairwise(expr.encode(), d, r, mode.encode(), a.ctypes.data_as(P),
                                  b.ctypes.data_as(P), res.ctypes.data_as(P), ctypes.c_int64(res.size),
                                  info, len(info)))
        res = res.reshape(rdims)
    return fa, costs, rdims, res


def layer(layer_json, cr=0.0):
    """Returns (expr, dims, param_count, ranks)."""
    import json
    out = _buf(1 << 16)
    _check(lib().ref_layer(layer_json.encode(), ctypes.c_double(cr), out, len(out)))
    expr, dims, pc, ranks = out.value.decode().split("\n")
    return expr, json.loads(dims), int(pc), [int(x) for x in ranks.split()]


def theorem_plan(layer_json, cost_mode="inference"):
    out = _buf()
    _check(lib().ref_theorem_plan(layer_json.encode(), cost_mode.encode(), out, len(out)))
    js, enc = out.value.decode().split("\n")
    return js, enc


def resnet34(batch, cr):
    out = _buf(1 << 16)
    _check(lib().ref_resnet34(ctypes.c_int64(batch), ctypes.c_double(cr), out, len(out)))
    rows = []
    for line in out.value.decode().strip().split("\n"):
        name, js = line.split(" ", 1)
        rows.append((name, js))
    return rows


def fill_random(shape, seed):
    shape = [int(s) for s in shape]
    out = np.zeros(max(1, int(np.prod(shape))), dtype=np.float64)
    arr = (ctypes.c_int64 * max(1, len(shape)))(*shape)
    _check(lib().ref_fill_random(arr, len(shape), ctypes.c_uint64(seed),
                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return out.reshape(shape)


def parse(expr):
    out = _buf(1 << 14)
    _check(lib().ref_parse(expr.encode(), out, len(out)))
    r, cls = out.value.decode().split("\n")
    return r, dict(x.split(":") for x in cls.split()) if cls else {}


def tensor_to_json(arr):
    a = np.ascontiguousarray(arr, dtype=np.float64)
    shp = (ctypes.c_int64 * max(1, a.ndim))(*a.shape)
    out = _buf(max(1 << 16, 32 * a.size + 256))
    _check(lib().ref_tensor_to_json(shp, a.ndim, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out, len(out)))
    return out.value.decode()


def tensor_from_json(text):
    shp = (ctypes.c_int64 * 64)()
    rank = ctypes.c_int()
    cnt = ctypes.c_int64()
    data = np.zeros(max(1, len(text)), dtype=np.float64)
    _check(lib().ref_tensor_from_json(text.encode(), shp, ctypes.byref(rank),
                                      data.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.c_int64(data.size),
                                      ctypes.byref(cnt)))
    return data[:cnt.value].reshape([shp[i] for i in range(rank.value)])


def tensor_to_binary(arr):
    a = np.ascontiguousarray(arr, dtype=np.float64)
    shp = (ctypes.c_int64 * max(1, a.ndim))(*a.shape)
    cap = 8 * (1 + a.ndim + a.size)
    out = ctypes.create_string_buffer(cap)
    ln = ctypes.c_int64()
    _check(lib().ref_tensor_to_binary(shp, a.ndim, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out,
                                      ctypes.c_int64(cap), ctypes.byref(ln)))
    return out.raw[:ln.value]


def layer_json_roundtrip(layer_json):
    out = _buf(1 << 12)
    _check(lib().ref_layer_json_roundtrip(layer_json.encode(), out, len(out)))
    return out.value.decode()


def merge_like_modes(expr1, dims, data):
    """Reference merge_like_modes + unmerge_modes on a one-input expression's classes:
    (permuted data, merged subs, merged dims, record, unmerged subs, unmerged dims)."""
    a = np.ascontiguousarray(data, dtype=np.float64)
    d = (ctypes.c_int64 * max(1, len(dims)))(*dims)
    out = np.zeros(max(1, a.size), dtype=np.float64)
    info = _buf(1 << 14)
    P = ctypes.POINTER(ctypes.c_double)
    _check(lib().ref_merge_like_modes(expr1.encode(), d, a.ctypes.data_as(P), out.ctypes.data_as(P), info, len(info)))
    ms, md, rec, us, ud = info.value.decode().split("\n")
    md = [int(x) for x in md.split(",")]
    return out[:a.size].reshape(md), ms, md, rec, us, [int(x) for x in ud.split(",")]
