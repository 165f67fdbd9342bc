"""Device executor bindings (torch tensors as device-memory plumbing only).

Context  -> ce_ctx   (one per GPU; work ordered on torch's current stream)
Executor -> ce_executor (plan compiled once into kernel steps + workspace)
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import torch

from . import _lib
from ._lib import check, lib
from .api import Plan, _dims_arg

MATH = {"auto": 0, "tf32": 0, "fp32": 1, "simt": 1, "3xtf32": 2}


class Context:
    """ce_ctx_create: binds a device and a stream (default: torch's current stream)."""

    def __init__(self, device: int = 0, math: str = "auto", stream: Optional[torch.cuda.Stream] = None,
                 graphs: bool = True):
        self.device = device
        self.math = math
        torch.cuda.set_device(device)
        st = stream if stream is not None else torch.cuda.current_stream(device)
        if st.cuda_stream == 0:
            # the legacy default stream has handle 0, which ce_ctx_create reads as "make your own";
            # use an explicit side stream instead so callers can order work on ctx.torch_stream
            st = torch.cuda.Stream(device)
        self.torch_stream = st
        opts = _lib.Options(MATH[math], int(graphs), ctypes.c_void_p(st.cuda_stream))
        h = ctypes.c_void_p()
        check(lib().ce_ctx_create(device, ctypes.byref(opts), ctypes.byref(h)))
        self._h = h
        self._destroy = lib().ce_ctx_destroy

    @property
    def handle(self):
        return self._h

    def synchronize(self):
        check(lib().ce_ctx_synchronize(self._h))

    def fill_random(self, shape: Sequence[int], seed: int) -> torch.Tensor:
        """fill_random (tensor.cpp:125-130) evaluated on the device, rounded to FP32."""
        cur = torch.cuda.current_stream(self.device)
        with torch.cuda.stream(self.torch_stream):
            t = torch.empty(list(shape), dtype=torch.float32, device=f"cuda:{self.device}")
            check(lib().ce_fill_random(self._h, ctypes.c_void_p(t.data_ptr()), t.numel(), ctypes.c_uint64(seed)))
        if cur.cuda_stream != self.torch_stream.cuda_stream:
            cur.wait_stream(self.torch_stream)
            t.record_stream(cur)
        return t

    # ------------------------------------------------------------ data parallel
    def init_comm(self, world: int, rank: int, unique_id: bytes):
        """Join an NCCL communicator of `world` contexts (ce_ctx_init_comm)."""
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        check(lib().ce_ctx_init_comm(self._h, world, rank, buf))
        self.has_comm = True

    def allreduce_grads(self, tensors: Sequence[torch.Tensor]):
        """In-place SUM all-reduce of FP32 device tensors on the context's comm stream
        (after the work queued on ctx.torch_stream); see comm_wait."""
        ts = [t for t in tensors if t is not None]
        if not ts:
            return
        self.torch_stream.wait_stream(torch.cuda.current_stream(self.device))
        ptrs = (ctypes.c_void_p * len(ts))(*[ctypes.c_void_p(t.data_ptr()) for t in ts])
        counts = (ctypes.c_int64 * len(ts))(*[t.numel() for t in ts])
        check(lib().ce_allreduce_grads(self._h, ptrs, counts, len(ts)))

    def comm_wait(self):
        """Order the context stream (and the caller's current stream) after the collectives."""
        check(lib().ce_comm_wait(self._h))
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream != self.torch_stream.cuda_stream:
            cur.wait_stream(self.torch_stream)

    def __del__(self):
        # the destroy entry point is bound at creation: module globals may be gone at exit
        if getattr(self, "_h", None) and getattr(self, "_destroy", None):
            self._destroy(self._h)
            self._h = None


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through libce (rank 0 creates it, every rank passes it to init_comm)."""
    buf = ctypes.create_string_buffer(128)
    check(lib().ce_nccl_unique_id(buf))
    return buf.raw


def _device_f32(ctx: Context, what: str, t: torch.Tensor) -> torch.Tensor:
    """A contiguous float32 tensor on the context's device (a copy when `t` is strided).
    The caller keeps the returned tensor alive until the library call that reads it returns
    and orders ctx.torch_stream after the caller's stream (where a copy is produced)."""
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float32:
        raise TypeError(f"{what} must be a float32 torch tensor")
    if not t.is_cuda or (t.device.index or 0) != ctx.device:
        raise TypeError(f"{what} must live on cuda:{ctx.device}")
    return t.contiguous()


def conv_einsum_forward(ctx: Context, expr: str, *tensors: torch.Tensor, mode: str = "same",
                        cost_mode: str = "inference") -> torch.Tensor:
    """ce_conv_einsum: plan + executor cached in the context by (expr, shapes, mode, cost_mode)."""
    from .api import Plan as _P
    # contiguous copies are made on the caller's stream and kept alive until the call returns
    ts = [_device_f32(ctx, f"input {i}", t) for i, t in enumerate(tensors)]
    dims = [list(t.shape) for t in ts]
    key = (expr, tuple(map(tuple, dims)), mode, cost_mode)
    shapes = ctx.__dict__.setdefault("_out_shapes", {})
    if key not in shapes:
        shapes[key] = _P.optimal(expr, dims, mode, cost_mode).out_dims
    ctx.torch_stream.wait_stream(torch.cuda.current_stream(ctx.device))
    out = torch.empty(shapes[key], dtype=torch.float32, device=ts[0].device)
    d, r, _ = _dims_arg(dims)
    ptrs = (ctypes.c_void_p * len(ts))(*[ctypes.c_void_p(t.data_ptr()) for t in ts])
    check(lib().ce_conv_einsum(ctx.handle, expr.encode(), d, r, len(ts), mode.encode(), cost_mode.encode(),
                               ctypes.cast(ptrs, _lib.c_fpp), ctypes.c_void_p(out.data_ptr())))
    cur = torch.cuda.current_stream(ctx.device)
    if cur.cuda_stream != ctx.torch_stream.cuda_stream:
        cur.wait_stream(ctx.torch_stream)
        for t in ts:
            t.record_stream(ctx.torch_stream)
    return out


def _ptrs(ts):
    arr = (ctypes.c_void_p * len(ts))(*[ctypes.c_void_p(t.data_ptr()) if t is not None else None for t in ts])
    return ctypes.cast(arr, _lib.c_fpp), arr


def _check_inputs(plan: Plan, inputs):
    if len(inputs) != plan.n_inputs:
        raise _lib.ShapeError(3, "execute: wrong number of input tensors")
    for i, (t, d) in enumerate(zip(inputs, plan.dims)):
        if list(t.shape) != list(d):
            raise _lib.ShapeError(3, f"execute: input {i} shape mismatch")
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
            raise TypeError(f"input {i} must be a contiguous CUDA float32 tensor")


class Executor:
    """execute() (sequencer.cpp:403-447) + backward on one device."""

    def __init__(self, ctx: Context, plan: Plan, backward: bool = False, recompute: bool = False):
        """recompute: gradient checkpointing -- backward() recomputes the
        forward intermediates instead of reading ones execute() kept."""
        from .api import CE_EXEC_RECOMPUTE
        self.ctx, self.plan = ctx, plan
        h = ctypes.c_void_p()
        wb = int(backward) | (CE_EXEC_RECOMPUTE if (backward and recompute) else 0)
        check(lib().ce_executor_create(ctx.handle, plan._h, wb, ctypes.byref(h)))
        self._h = h
        self._destroy = lib().ce_executor_destroy
        self.stats = _lib.ExecStats()

    def _order_in(self):
        """Make the ctx stream wait for the caller's current stream (inputs produced there)."""
        cur = torch.cuda.current_stream(self.ctx.device)
        if cur.cuda_stream != self.ctx.torch_stream.cuda_stream:
            self.ctx.torch_stream.wait_stream(cur)
            return cur
        return None

    def _order_out(self, cur, tensors):
        if cur is not None:
            cur.wait_stream(self.ctx.torch_stream)
            for t in tensors:
                if t is not None:
                    t.record_stream(cur)

    def execute(self, inputs: Sequence[torch.Tensor], out: Optional[torch.Tensor] = None) -> torch.Tensor:
        _check_inputs(self.plan, inputs)
        cur = self._order_in()
        with torch.cuda.stream(self.ctx.torch_stream):
            if out is None:
                out = torch.empty(self.plan.out_dims, dtype=torch.float32, device=inputs[0].device)
            p, keep = _ptrs(list(inputs))
            check(lib().ce_execute(self._h, p, ctypes.c_void_p(out.data_ptr()), ctypes.byref(self.stats)))
            del keep
        self._order_out(cur, [out])
        return out

    def backward(self, inputs: Sequence[torch.Tensor], dout: torch.Tensor,
                 needs: Optional[Sequence[bool]] = None) -> List[Optional[torch.Tensor]]:
        _check_inputs(self.plan, inputs)
        needs = needs or [True] * len(inputs)
        cur = self._order_in()
        with torch.cuda.stream(self.ctx.torch_stream):
            grads = [torch.empty_like(t) if n else None for t, n in zip(inputs, needs)]
            p, k1 = _ptrs(list(inputs))
            g, k2 = _ptrs(grads)
            dout = dout.contiguous()
            check(lib().ce_backward(self._h, p, ctypes.c_void_p(dout.data_ptr()), g, ctypes.byref(self.stats)))
            del k1, k2
        self._order_out(cur, grads)
        return grads

    def set_profiling(self, on: bool = True):
        check(lib().ce_executor_set_profiling(self._h, int(on)))

    def profile(self, backward: bool = False):
        """[(label, kind, ms, flops, bytes)] of the last forward/backward call (CUDA events per kernel)."""
        n_max = 256
        n = ctypes.c_int()
        labels = ctypes.create_string_buffer(1 << 16)
        kinds = (ctypes.c_int * n_max)()
        ms = (ctypes.c_float * n_max)()
        fl = (ctypes.c_double * n_max)()
        by = (ctypes.c_double * n_max)()
        check(lib().ce_executor_profile(self._h, int(backward), n_max, ctypes.byref(n), labels, len(labels), kinds,
                                        ms, fl, by))
        names = labels.value.decode().split("\n")
        kind_names = ["direct", "tiled", "tc", "memset", "reduce", "permute", "fused", "split", "pconv", "row"]
        return [(names[i], kind_names[kinds[i]], float(ms[i]), float(fl[i]), float(by[i])) for i in range(n.value)]

    def execute_host(self, host_inputs: Sequence["numpy.ndarray"], host_out: "numpy.ndarray"):  # noqa: F821
        """H2D + execute + D2H + sync through the C-ABI (the end-to-end call)."""
        arrs = [a for a in host_inputs]
        ptrs = (ctypes.c_void_p * len(arrs))(*[ctypes.c_void_p(a.ctypes.data) for a in arrs])
        check(lib().ce_execute_host(self._h, ctypes.cast(ptrs, _lib.c_fpp), ctypes.c_void_p(host_out.ctypes.data)))

    def __del__(self):
        # the destroy entry point is bound at creation: module globals may be gone at exit
        if getattr(self, "_h", None) and getattr(self, "_destroy", None):
            self._destroy(self._h)
            self._h = None


def pairwise_eval(ctx: Context, expr: str, a: torch.Tensor, b: torch.Tensor, mode: str = "same") -> torch.Tensor:
    """pairwise_eval (kernels.cpp:425-470) for expr "L,R->RES|convs" (keep = RES, order RES)."""
    from .api import Plan as _P  # result shape via a one-node plan
    a, b = _device_f32(ctx, "a", a), _device_f32(ctx, "b", b)
    shape = _P.optimal(expr, [list(a.shape), list(b.shape)], mode).out_dims
    ctx.torch_stream.wait_stream(torch.cuda.current_stream(ctx.device))  # ce_pairwise_* syncs its own stream
    out = torch.empty(shape, dtype=torch.float32, device=a.device)
    d, r, _ = _dims_arg([list(a.shape), list(b.shape)])
    check(lib().ce_pairwise_eval(ctx.handle, expr.encode(), d, r, mode.encode(), ctypes.c_void_p(a.data_ptr()),
                                 ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(out.data_ptr())))
    return out


def pairwise_grad(ctx: Context, expr: str, a, b, dout, mode: str = "same"):
    """Adjoints (dA, dB) of <dout, pairwise_eval(a, b)> (ce_pairwise_grad)."""
    from .api import Plan as _P
    a, b, dout = _device_f32(ctx, "a", a), _device_f32(ctx, "b", b), _device_f32(ctx, "dout", dout)
    shape = _P.optimal(expr, [list(a.shape), list(b.shape)], mode).out_dims
    if list(dout.shape) != list(shape):
        raise _lib.ShapeError(3, f"pairwise_grad: dout shape {list(dout.shape)} != result shape {list(shape)}")
    ctx.torch_stream.wait_stream(torch.cuda.current_stream(ctx.device))
    da, db = torch.empty_like(a), torch.empty_like(b)
    d, r, _ = _dims_arg([list(a.shape), list(b.shape)])
    check(lib().ce_pairwise_grad(ctx.handle, expr.encode(), d, r, mode.encode(), ctypes.c_void_p(a.data_ptr()),
                                 ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(dout.data_ptr()),
                                 ctypes.c_void_p(da.data_ptr()), ctypes.c_void_p(db.data_ptr())))
    return da, db


# ----------------------------------------------------------------------------- autograd
_PLAN_CACHE: dict = {}
_CTX_CACHE: dict = {}


def _context(device: int, math: str) -> Context:
    key = (device, math, torch.cuda.current_stream(device).cuda_stream)
    if key not in _CTX_CACHE:
        _CTX_CACHE[key] = Context(device, math)
    return _CTX_CACHE[key]


def _executor(expr, shapes, mode, cost_mode, device, math):
    key = (expr, tuple(tuple(s) for s in shapes), mode, cost_mode, device, math)
    if key not in _PLAN_CACHE:
        plan = Plan.optimal(expr, shapes, mode, cost_mode)
        _PLAN_CACHE[key] = Executor(_context(device, math), plan, backward=True)
    return _PLAN_CACHE[key]


class _ConvEinsumFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, expr, mode, math, *tensors):
        ts = [t.contiguous() for t in tensors]
        ex = _executor(expr, [list(t.shape) for t in ts], mode, "training", ts[0].device.index or 0, math)
        out = ex.execute(ts)
        ctx.ex = ex
        ctx.save_for_backward(*ts)
        return out

    @staticmethod
    def backward(ctx, dout):
        ts = ctx.saved_tensors
        # the executor's workspace holds the intermediates of its LAST forward; another
        # call may have run since, so recompute them for these inputs
        ctx.ex.execute(list(ts))
        grads = ctx.ex.backward(list(ts), dout.contiguous(), list(ctx.needs_input_grad[3:]))
        return (None, None, None, *grads)


def conv_einsum(expr: str, *tensors: torch.Tensor, mode: str = "same", math: str = "auto") -> torch.Tensor:
    """The paper's call form conv_einsum("...", T1, T2, ...), differentiable."""
    return _ConvEinsumFn.apply(expr, mode, math, *tensors)


# ----------------------------------------------------------------------------- like-mode merging
def merge_like_modes(ctx: Context, t: torch.Tensor, subs: str, classes: dict):
    """merge_like_modes (kernels.hpp:88-94) on the device: returns (merged tensor, merged
    subscripts, record).  `classes`: atom -> class name as api.classify() returns."""
    if not (t.is_cuda and t.dtype == torch.float32):
        raise TypeError("merge_like_modes: a CUDA float32 tensor")
    t = t.contiguous()
    d = (ctypes.c_int64 * max(1, t.dim()))(*t.shape)
    cls = " ".join(f"{a}:{c}" for a, c in classes.items()).encode()
    out = torch.empty_like(t)
    ms = ctypes.create_string_buffer(1024)
    md = (ctypes.c_int64 * 64)()
    mr = ctypes.c_int()
    rec = ctypes.create_string_buffer(4096)
    cur = torch.cuda.current_stream(t.device)
    ctx.torch_stream.wait_stream(cur)
    check(lib().ce_merge_like_modes(ctx.handle, subs.encode(), d, cls, ctypes.c_void_p(t.data_ptr()),
                                    ctypes.c_void_p(out.data_ptr()), ms, len(ms), md, ctypes.byref(mr), rec,
                                    len(rec)))
    cur.wait_stream(ctx.torch_stream)
    t.record_stream(ctx.torch_stream)
    out.record_stream(cur)
    return out.view([int(md[i]) for i in range(mr.value)]), ms.value.decode(), rec.value.decode()


def unmerge_modes(t: torch.Tensor, subs: str, record: str):
    """unmerge_modes (kernels.hpp:96-98): a reshape back to the member axes."""
    d = (ctypes.c_int64 * max(1, t.dim()))(*t.shape)
    us = ctypes.create_string_buffer(1024)
    ud = (ctypes.c_int64 * 64)()
    ur = ctypes.c_int()
    check(lib().ce_unmerge_modes(subs.encode(), d, record.encode(), us, len(us), ud, ctypes.byref(ur)))
    return t.view([int(ud[i]) for i in range(ur.value)]), us.value.decode()
