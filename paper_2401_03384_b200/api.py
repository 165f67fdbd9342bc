"""Python mirror of the reference `convexpr` API for the executor path.

Names and argument meaning follow /root/reference/proj/include/convexpr:
  parse/render/classify          expression.hpp:76-83
  optimal/left_to_right/...      sequencer.hpp:44-95  (here: Plan.optimal(...) etc.)
  execute                        sequencer.hpp:88     (here: Executor.execute)
  pairwise_eval                  kernels.hpp:105
  expression / rank_for_compression / resnet34_cp_blocks   layers.hpp:71-94
Errors raise ParseError / ShapeError / PlanError like the reference's exceptions.
All device work goes through libce.so (include/ce/ce.h); tensors are torch CUDA
float32 tensors used purely as device-memory plumbing.
"""
from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass, field
from typing import Optional, Sequence

from . import _lib
from ._lib import CeError, ParseError, PlanError, ShapeError, check, lib  # noqa: F401

MODES = ("full", "same", "valid", "circular")


CE_EXEC_RECOMPUTE = 0x100  # include/ce/ce.h: gradient checkpointing flag of want_backward


def _dims_arg(dims: Sequence[Sequence[int]]):
    flat = [int(d) for ds in dims for d in ds]
    ranks = [len(ds) for ds in dims]
    return (ctypes.c_int64 * max(1, len(flat)))(*flat), (ctypes.c_int * max(1, len(ranks)))(*ranks), len(ranks)


def _u128(lo, hi):
    return int(lo) | (int(hi) << 64)


# ----------------------------------------------------------------------------- IR
@dataclass
class Spec:
    rendered: str
    classes: dict


def parse(expr: str) -> Spec:
    """parse + render + classify; raises ParseError with the byte position."""
    r = ctypes.create_string_buffer(1 << 14)
    c = ctypes.create_string_buffer(1 << 14)
    check(lib().ce_parse(expr.encode(), r, len(r), c, len(c)))
    cls = dict(x.split(":") for x in c.value.decode().split()) if c.value else {}
    return Spec(r.value.decode(), cls)


def render(expr: str) -> str:
    return parse(expr).rendered


def classify(expr: str) -> dict:
    return parse(expr).classes


# ----------------------------------------------------------------------------- plans
@dataclass
class PlanNodeInfo:
    left: int
    right: int
    result: str
    flops_actual: int
    cost: int


class Plan:
    """An EvaluationPlan (sequencer.hpp:30-41) held by libce."""

    def __init__(self, handle, expr, dims, mode, cost_mode):
        self._h = handle
        self._destroy = lib().ce_plan_destroy
        self.expr, self.dims, self.mode, self.cost_mode = expr, [list(map(int, d)) for d in dims], mode, cost_mode
        info = _lib.PlanInfo()
        check(lib().ce_plan_get_info(self._h, ctypes.byref(info)))
        self.n_inputs = info.n_inputs
        self.n_nodes = info.n_nodes
        self.out_dims = [int(info.out_dims[i]) for i in range(info.out_rank)]
        self.total_cost = _u128(info.total_cost_lo, info.total_cost_hi)
        self.inference_cost = _u128(info.inference_cost_lo, info.inference_cost_hi)
        self.training_cost = _u128(info.training_cost_lo, info.training_cost_hi)
        self.flops_actual = _u128(info.flops_actual_lo, info.flops_actual_hi)
        self.peak_intermediate_elements = int(info.peak_intermediate_elements)

    @staticmethod
    def _create(expr, dims, mode, cost_mode, strategy):
        d, r, n = _dims_arg(dims)
        h = ctypes.c_void_p()
        check(lib().ce_plan_create(expr.encode(), d, r, n, mode.encode(), cost_mode.encode(), strategy, ctypes.byref(h)))
        return Plan(h, expr, dims, mode, cost_mode)

    @classmethod
    def optimal(cls, expr, dims, mode="same", cost_mode="inference", cost_capped=False):
        return cls._create(expr, dims, mode, cost_mode, 2 if cost_capped else 0)

    @classmethod
    def left_to_right(cls, expr, dims, mode="same", cost_mode="inference"):
        return cls._create(expr, dims, mode, cost_mode, 1)

    @classmethod
    def from_joins(cls, expr, dims, joins, mode="same", cost_mode="inference"):
        d, r, n = _dims_arg(dims)
        flat = [int(x) for j in joins for x in j]
        arr = (ctypes.c_int * max(1, len(flat)))(*flat)
        h = ctypes.c_void_p()
        check(lib().ce_plan_from_joins(expr.encode(), d, r, n, mode.encode(), cost_mode.encode(), arr, len(joins),
                                       ctypes.byref(h)))
        return Plan(h, expr, dims, mode, cost_mode)

    @classmethod
    def from_nodes(cls, expr, dims, nodes, mode="same", cost_mode="inference"):
        """Replay a caller's plan: nodes = [(left id, right id, result subscripts)] (plan_to_json's
        node fields); mode may be a per-atom map "h=same,w=circular"."""
        d, r, n = _dims_arg(dims)
        flat = [int(x) for (l, rr, _) in nodes for x in (l, rr)]
        arr = (ctypes.c_int * max(1, len(flat)))(*flat)
        res = (ctypes.c_char_p * max(1, len(nodes)))(*[str(x[2]).encode() for x in nodes])
        h = ctypes.c_void_p()
        check(lib().ce_plan_from_nodes(expr.encode(), d, r, n, mode.encode(), cost_mode.encode(), arr, res,
                                       len(nodes), ctypes.byref(h)))
        return Plan(h, expr, dims, mode, cost_mode)

    def to_json(self) -> str:
        buf = ctypes.create_string_buffer(1 << 20)
        check(lib().ce_plan_json(self._h, buf, len(buf)))
        return buf.value.decode()

    def tree_encoding(self) -> str:
        buf = ctypes.create_string_buffer(1 << 16)
        check(lib().ce_plan_tree_encoding(self._h, buf, len(buf)))
        return buf.value.decode()

    def describe_steps(self, backward: bool = False, math: str = "auto", recompute: bool = False) -> str:
        """Kernel steps the device executor compiles this plan into (no GPU needed)."""
        buf = ctypes.create_string_buffer(1 << 20)
        wb = int(backward) | (CE_EXEC_RECOMPUTE if recompute else 0)
        check(lib().ce_plan_describe_steps(self._h, wb, {"auto": 0, "tf32": 0, "3xtf32": 2}.get(math, 1), buf, len(buf)))
        return buf.value.decode()

    def nodes(self):
        out = []
        for j in range(self.n_nodes):
            l, r = ctypes.c_int(), ctypes.c_int()
            buf = ctypes.create_string_buffer(4096)
            fa, cost = ctypes.c_uint64(), ctypes.c_uint64()
            check(lib().ce_plan_node(self._h, j, ctypes.byref(l), ctypes.byref(r), buf, len(buf), ctypes.byref(fa),
                                     ctypes.byref(cost)))
            out.append(PlanNodeInfo(l.value, r.value, buf.value.decode(), fa.value, cost.value))
        return out

    def __del__(self):
        # the destroy entry point is bound at creation: module globals may be gone at exit
        if getattr(self, "_h", None) and getattr(self, "_destroy", None):
            self._destroy(self._h)
            self._h = None


def optimal(expr, dims, mode="same", cost_mode="inference", cost_capped=False) -> Plan:
    return Plan.optimal(expr, dims, mode, cost_mode, cost_capped)


def left_to_right(expr, dims, mode="same", cost_mode="inference") -> Plan:
    return Plan.left_to_right(expr, dims, mode, cost_mode)


def plan_from_joins(expr, dims, joins, mode="same", cost_mode="inference") -> Plan:
    return Plan.from_joins(expr, dims, joins, mode, cost_mode)


def plan_from_nodes(expr, dims, nodes, mode="same", cost_mode="inference") -> Plan:
    return Plan.from_nodes(expr, dims, nodes, mode, cost_mode)


def plan_to_json(plan: Plan) -> str:
    return plan.to_json()


def tree_encoding(plan: Plan) -> str:
    return plan.tree_encoding()


# ----------------------------------------------------------------------------- layers
@dataclass
class LayerSpec:
    """layers.hpp:46-58 (channel factors, filter H/W, feature H'/W', batch, ranks)."""
    kind: str = "standard"
    t_factors: list = field(default_factory=lambda: [1])
    s_factors: list = field(default_factory=lambda: [1])
    filter_h: int = 3
    filter_w: int = 3
    feature_h: int = 32
    feature_w: int = 32
    batch: int = 1
    ranks: list = field(default_factory=list)

    @staticmethod
    def from_json(text: str) -> "LayerSpec":
        """layer_from_json (layers.cpp:448-467) field names."""
        j = json.loads(text)
        lst = lambda v: list(v) if isinstance(v, list) else [v]  # noqa: E731
        r = lst(j["rank"]) if "rank" in j else []
        return LayerSpec(j["kind"], lst(j["T"]), lst(j["S"]), j["H"], j["W"], j["Hp"], j["Wp"], j.get("B", 1), r)


@dataclass
class LayerExpression:
    expr: str
    dims: list
    ranks: list
    param_count: int


def expression(layer: LayerSpec, cr: Optional[float] = None) -> LayerExpression:
    """expression() (layers.cpp:147-327); with cr, ranks from rank_for_compression first."""
    t = (ctypes.c_int64 * len(layer.t_factors))(*layer.t_factors)
    s = (ctypes.c_int64 * len(layer.s_factors))(*layer.s_factors)
    rk = list(layer.ranks) or [1]
    r = (ctypes.c_int64 * len(rk))(*rk)
    ebuf = ctypes.create_string_buffer(1 << 14)
    dims = (ctypes.c_int64 * 256)()
    rofi = (ctypes.c_int * 32)()
    nin = ctypes.c_int()
    rout = (ctypes.c_int64 * 32)()
    nrout = ctypes.c_int()
    pc = ctypes.c_uint64()
    check(lib().ce_layer_expression(layer.kind.encode(), t, len(layer.t_factors), s, len(layer.s_factors),
                                    layer.filter_h, layer.filter_w, layer.feature_h, layer.feature_w, layer.batch, r,
                                    len(layer.ranks), ctypes.c_double(cr or 0.0), ebuf, len(ebuf), dims, 256, rofi,
                                    ctypes.byref(nin), rout, ctypes.byref(nrout), ctypes.byref(pc)))
    out, pos = [], 0
    for i in range(nin.value):
        out.append([int(dims[pos + k]) for k in range(rofi[i])])
        pos += rofi[i]
    return LayerExpression(ebuf.value.decode(), out, [int(rout[i]) for i in range(nrout.value)], int(pc.value))


def flops_actual(expr: str, dims: Sequence[Sequence[int]], mode: str = "same") -> int:
    """flops_actual (kernels.cpp:472-505) of the pairwise op "L,R->RES|convs" (exact MACs)."""
    d, r, _ = _dims_arg(dims)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib().ce_flops_actual(expr.encode(), d, r, mode.encode(), ctypes.byref(lo), ctypes.byref(hi)))
    return _u128(lo.value, hi.value)


def rank_for_compression(layer: LayerSpec, cr: float) -> int:
    return expression(layer, cr).ranks[0]


RESNET34_STAGES = [("conv1", 3, 64, 7, 112), ("conv2_x", 64, 64, 3, 56), ("conv3_x", 128, 128, 3, 28),
                   ("conv4_x", 256, 256, 3, 14), ("conv5_x", 512, 512, 3, 7)]


def resnet34_cp_blocks(batch: int, cr: float):
    """resnet34_cp_blocks (layers.cpp:400-423)."""
    out = []
    for name, s, t, k, feat in RESNET34_STAGES:
        l = LayerSpec("cp", [t], [s], k, k, feat, feat, batch, [1])
        l.ranks = [rank_for_compression(l, cr)]
        out.append((name, l))
    return out
