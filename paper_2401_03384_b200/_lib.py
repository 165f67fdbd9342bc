"""ctypes binding of include/ce/ce.h (libce.so, built in-tree by csrc/Makefile).

There is no fallback: if libce.so is missing or fails to load, importing the
package raises.  The product path never touches oracle/.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CE_LIB_PATH: an alternate build of the same library for same-box A/B experiments
LIB_PATH = os.environ.get("CE_LIB_PATH") or os.path.join(_HERE, "libce.so")

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_intp = ctypes.POINTER(ctypes.c_int)
c_fp = ctypes.POINTER(ctypes.c_float)
c_fpp = ctypes.POINTER(ctypes.c_void_p)


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_inputs", ctypes.c_int), ("n_nodes", ctypes.c_int), ("out_rank", ctypes.c_int),
        ("out_dims", ctypes.c_int64 * 16),
        ("total_cost_lo", ctypes.c_uint64), ("total_cost_hi", ctypes.c_uint64),
        ("inference_cost_lo", ctypes.c_uint64), ("inference_cost_hi", ctypes.c_uint64),
        ("training_cost_lo", ctypes.c_uint64), ("training_cost_hi", ctypes.c_uint64),
        ("flops_actual_lo", ctypes.c_uint64), ("flops_actual_hi", ctypes.c_uint64),
        ("peak_intermediate_elements", ctypes.c_uint64),
    ]


class Options(ctypes.Structure):
    _fields_ = [("math", ctypes.c_int), ("use_graphs", ctypes.c_int), ("stream", ctypes.c_void_p)]


class ExecStats(ctypes.Structure):
    _fields_ = [
        ("multiplications_lo", ctypes.c_uint64), ("multiplications_hi", ctypes.c_uint64),
        ("peak_intermediate_elements", ctypes.c_uint64),
        ("kernels_launched", ctypes.c_int), ("tc_steps", ctypes.c_int),
    ]


# Every exported symbol of include/ce/ce.h with its ctypes signature.
SIGNATURES = {
    "ce_last_error": (ctypes.c_char_p, []),
    "ce_version": (ctypes.c_char_p, []),
    "ce_parse": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]),
    "ce_plan_create": (ctypes.c_int, [ctypes.c_char_p, c_i64p, c_intp, ctypes.c_int, ctypes.c_char_p,
                                      ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "ce_plan_from_joins": (ctypes.c_int, [ctypes.c_char_p, c_i64p, c_intp, ctypes.c_int, ctypes.c_char_p,
                                          ctypes.c_char_p, c_intp, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "ce_plan_from_nodes": (ctypes.c_int, [ctypes.c_char_p, c_i64p, c_intp, ctypes.c_int, ctypes.c_char_p,
                                          ctypes.c_char_p, c_intp, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int,
                                          ctypes.POINTER(ctypes.c_void_p)]),
    "ce_plan_destroy": (None, [ctypes.c_void_p]),
    "ce_plan_json": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]),
    "ce_plan_tree_encoding": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t]),
    "ce_plan_get_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PlanInfo)]),
    "ce_plan_node": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, c_intp, c_intp, ctypes.c_char_p, ctypes.c_size_t,
                                    ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]),
    "ce_plan_describe_steps": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                              ctypes.c_size_t]),
    "ce_layer_expression": (ctypes.c_int, [ctypes.c_char_p, c_i64p, ctypes.c_int, c_i64p, ctypes.c_int,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int64, c_i64p, ctypes.c_int, ctypes.c_double, ctypes.c_char_p,
                                           ctypes.c_size_t, c_i64p, ctypes.c_int, c_intp, c_intp, c_i64p, c_intp,
                                           ctypes.POINTER(ctypes.c_uint64)]),
    "ce_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(Options), ctypes.POINTER(ctypes.c_void_p)]),
    "ce_ctx_destroy": (None, [ctypes.c_void_p]),
    "ce_ctx_stream": (ctypes.c_void_p, [ctypes.c_void_p]),
    "ce_ctx_synchronize": (ctypes.c_int, [ctypes.c_void_p]),
    "ce_ctx_workspace_bytes": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]),
    "ce_ctx_alloc": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "ce_ctx_free": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "ce_ctx_memcpy": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "ce_fill_random": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64]),
    "ce_executor_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "ce_executor_destroy": (None, [ctypes.c_void_p]),
    "ce_execute": (ctypes.c_int, [ctypes.c_void_p, c_fpp, ctypes.c_void_p, ctypes.POINTER(ExecStats)]),
    "ce_backward": (ctypes.c_int, [ctypes.c_void_p, c_fpp, ctypes.c_void_p, c_fpp, ctypes.POINTER(ExecStats)]),
    "ce_execute_host": (ctypes.c_int, [ctypes.c_void_p, c_fpp, ctypes.c_void_p]),
    "ce_executor_set_profiling": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "ce_executor_profile": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, c_intp, ctypes.c_char_p,
                                           ctypes.c_size_t, c_intp, ctypes.POINTER(ctypes.c_float),
                                           ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "ce_pairwise_eval": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, c_i64p, c_intp, ctypes.c_char_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "ce_pairwise_grad": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, c_i64p, c_intp, ctypes.c_char_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p]),
    "ce_flops_actual": (ctypes.c_int, [ctypes.c_char_p, c_i64p, c_intp, ctypes.c_char_p,
                                       ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]),
    "ce_conv_einsum": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, c_i64p, c_intp, ctypes.c_int,
                                      ctypes.c_char_p, ctypes.c_char_p, c_fpp, ctypes.c_void_p]),
    "ce_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "ce_ctx_init_comm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]),
    "ce_allreduce_grads": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p), c_i64p, ctypes.c_int]),
    "ce_comm_wait": (ctypes.c_int, [ctypes.c_void_p]),
    "ce_comm_check": (ctypes.c_int, [ctypes.c_void_p]),
    "ce_merge_like_modes": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, c_i64p, ctypes.c_char_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_char_p, ctypes.c_size_t, c_i64p, c_intp,
                                           ctypes.c_char_p, ctypes.c_size_t]),
    "ce_unmerge_modes": (ctypes.c_int, [ctypes.c_char_p, c_i64p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t,
                                        c_i64p, c_intp]),
    "ce_tensor_to_json": (ctypes.c_int, [c_i64p, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_char_p,
                                         ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "ce_tensor_from_json": (ctypes.c_int, [ctypes.c_char_p, c_i64p, ctypes.c_int, c_intp,
                                           ctypes.POINTER(ctypes.c_double), ctypes.c_int64, c_i64p]),
    "ce_tensor_to_binary": (ctypes.c_int, [c_i64p, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.c_char_p,
                                           ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "ce_tensor_from_binary": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, c_i64p, ctypes.c_int, c_intp,
                                             ctypes.POINTER(ctypes.c_double), ctypes.c_int64, c_i64p]),
    "ce_layer_to_json": (ctypes.c_int, [ctypes.c_char_p, c_i64p, ctypes.c_int, c_i64p, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, c_i64p,
                                        ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]),
    "ce_layer_from_json": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t, c_i64p, c_intp, c_i64p,
                                          c_intp, c_i64p, c_i64p, c_intp]),
}

STATUS = {0: "OK", 1: "OTHER", 2: "PARSE", 3: "SHAPE", 4: "NUMERIC", 5: "PLAN", 6: "OVERFLOW",
          7: "CUDA", 8: "NCCL", 9: "UNSUPPORTED"}


class CeError(RuntimeError):
    """Carries the ce_status code; subclasses mirror the reference exception types."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class ParseError(CeError):
    pass


class ShapeError(CeError):
    pass


class PlanError(CeError):
    pass


class OverflowError_(CeError):
    pass


_BY_CODE = {2: ParseError, 3: ShapeError, 5: PlanError, 6: OverflowError_}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libce.so not built at {LIB_PATH}: run `make -C paper_2401_03384_b200/csrc` "
                              "or __graft_entry__.build() (there is no CPU fallback)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def check(code: int):
    if code != 0:
        msg = lib().ce_last_error().decode()
        raise _BY_CODE.get(code, CeError)(code, msg)
