"""B200-native conv_einsum executor (arXiv 2401.03384).

Host planner (parse / optimal / layers) and the sm_100a device executor live in
libce.so behind include/ce/ce.h; this package is a thin ctypes mirror of the
reference `convexpr` API.  Importing it loads libce.so and fails loudly if it
is missing — there is no CPU fallback.
"""
from . import _lib
from .api import (CeError, LayerExpression, LayerSpec, ParseError, Plan, PlanError, ShapeError,  # noqa: F401
                  classify, expression, flops_actual, left_to_right, optimal, parse, plan_from_joins, plan_from_nodes, plan_to_json,
                  rank_for_compression, render, resnet34_cp_blocks, tree_encoding)

_lib.lib()  # load now: no silent fallback

__all__ = ["parse", "render", "classify", "optimal", "left_to_right", "plan_from_joins", "plan_from_nodes", "plan_to_json",
           "tree_encoding", "Plan", "LayerSpec", "LayerExpression", "expression", "rank_for_compression",
           "resnet34_cp_blocks", "flops_actual", "ParseError", "ShapeError", "PlanError", "CeError"]


def __getattr__(name):
    # device layer is imported lazily so planner-only users need no torch.cuda
    if name in ("Context", "Executor", "pairwise_eval", "pairwise_grad", "conv_einsum", "conv_einsum_forward",
                "nccl_unique_id"):
        from . import device
        return getattr(device, name)
    raise AttributeError(name)
