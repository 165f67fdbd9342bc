"""Wire formats through libce's C-ABI: the reference's tensor JSON / binary
serialisation (tensor.cpp:132-186, FP64 payload as DenseTensor holds it) and the layer
descriptor JSON (layers.cpp:425-467).  plan_to_json is api.plan_to_json."""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import check, lib
from .api import LayerSpec

_DP = ctypes.POINTER(ctypes.c_double)


def _shape_arg(shape):
    shape = [int(d) for d in shape]
    return (ctypes.c_int64 * max(1, len(shape)))(*shape), len(shape)


def tensor_to_json(t: np.ndarray) -> str:
    """tensor_to_json (tensor.cpp:132-137)."""
    a = np.ascontiguousarray(t, dtype=np.float64)
    sh, r = _shape_arg(a.shape)
    n = ctypes.c_size_t()
    lib().ce_tensor_to_json(sh, r, a.ctypes.data_as(_DP), None, 0, ctypes.byref(n))  # size query
    buf = ctypes.create_string_buffer(n.value)
    check(lib().ce_tensor_to_json(sh, r, a.ctypes.data_as(_DP), buf, len(buf), ctypes.byref(n)))
    return buf.value.decode()


def tensor_from_json(text: str) -> np.ndarray:
    """tensor_from_json (tensor.cpp:139-147): ParseError / ShapeError as the reference."""
    sh = (ctypes.c_int64 * 64)()
    rank = ctypes.c_int()
    count = ctypes.c_int64()
    raw = text.encode()
    lib().ce_tensor_from_json(raw, sh, 64, ctypes.byref(rank), None, 0, ctypes.byref(count))  # size query
    data = np.zeros(max(1, count.value), dtype=np.float64)
    check(lib().ce_tensor_from_json(raw, sh, 64, ctypes.byref(rank), data.ctypes.data_as(_DP), data.size,
                                    ctypes.byref(count)))
    return data[:count.value].reshape([int(sh[i]) for i in range(rank.value)])


def tensor_to_binary(t: np.ndarray) -> bytes:
    """tensor_write_binary (tensor.cpp:149-160): u64 rank, u64 dims, f64 payload, little-endian."""
    a = np.ascontiguousarray(t, dtype=np.float64)
    sh, r = _shape_arg(a.shape)
    n = 8 * (1 + a.ndim + a.size)
    buf = ctypes.create_string_buffer(n)
    ln = ctypes.c_size_t()
    check(lib().ce_tensor_to_binary(sh, r, a.ctypes.data_as(_DP), buf, n, ctypes.byref(ln)))
    return buf.raw[:ln.value]


def tensor_from_binary(raw: bytes) -> np.ndarray:
    """tensor_read_binary (tensor.cpp:162-173)."""
    sh = (ctypes.c_int64 * 64)()
    rank = ctypes.c_int()
    count = ctypes.c_int64()
    data = np.zeros(max(1, len(raw) // 8), dtype=np.float64)
    check(lib().ce_tensor_from_binary(raw, len(raw), sh, 64, ctypes.byref(rank), data.ctypes.data_as(_DP), data.size,
                                      ctypes.byref(count)))
    return data[:count.value].reshape([int(sh[i]) for i in range(rank.value)])


def layer_to_json(layer: LayerSpec) -> str:
    """layer_to_json (layers.cpp:425-440)."""
    t = (ctypes.c_int64 * len(layer.t_factors))(*layer.t_factors)
    s = (ctypes.c_int64 * len(layer.s_factors))(*layer.s_factors)
    r = (ctypes.c_int64 * max(1, len(layer.ranks)))(*layer.ranks)
    buf = ctypes.create_string_buffer(4096)
    check(lib().ce_layer_to_json(layer.kind.encode(), t, len(layer.t_factors), s, len(layer.s_factors),
                                 layer.filter_h, layer.filter_w, layer.feature_h, layer.feature_w, layer.batch, r,
                                 len(layer.ranks), buf, len(buf)))
    return buf.value.decode()


def layer_from_json(text: str) -> LayerSpec:
    """layer_from_json (layers.cpp:442-467), incl. validate()."""
    kind = ctypes.create_string_buffer(64)
    t, s, r = (ctypes.c_int64 * 32)(), (ctypes.c_int64 * 32)(), (ctypes.c_int64 * 32)()
    nt, ns, nr = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    hw = (ctypes.c_int64 * 5)()
    check(lib().ce_layer_from_json(text.encode(), kind, len(kind), t, ctypes.byref(nt), s, ctypes.byref(ns), hw, r,
                                   ctypes.byref(nr)))
    return LayerSpec(kind.value.decode(), list(t[:nt.value]), list(s[:ns.value]), int(hw[0]), int(hw[1]), int(hw[2]),
                     int(hw[3]), int(hw[4]), list(r[:nr.value]))
