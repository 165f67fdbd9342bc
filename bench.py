"""Benchmark: tensorized 3x3 conv layers (Tucker + TT, cfg2 of BASELINE.json),
batch 128 per GPU, 256->256 channels, 14x14, forward + backward on B200.

One step = forward + backward (input AND factor gradients) of four layers
  TK cr=0.1 (R=57), TK cr=1.0 (R=229), TT cr=0.1 (R=65), TT cr=1.0 (R=273)
through libce's C-ABI (plans from the reference-identical planner, training
cost mode).  `value` = algorithmic TFLOP/s over all GPUs = sum over nodes of
2*flops_actual (forward) + 2*flops_actual per adjoint (dA, dB), divided by the
device time of the step (CUDA events on the executor stream, max over ranks).
L2 is flushed (256 MiB write) between timed steps, outside the events.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--no-cfg3]

Multi-GPU: one process per GPU (torchrun; `--gpus N` without RANK in the environment
re-launches itself under torch.distributed.run), batch sharded (128 per GPU, weak
scaling), factors replicated, factor gradients all-reduced with NCCL.

`--impl reference` times the reference's own CPU executor (the unmodified convexpr
sources compiled by oracle/Makefile into oracle/_ref, FP64, OpenMP on every host core)
on a bounded batch sample of the same four layers; everything it reports (expression,
ranks, plan, executed multiplications) comes from that library, not from libce.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LAYERS = [("tk", 0.1), ("tk", 1.0), ("tt", 0.1), ("tt", 1.0)]
SLOTS = {"tk": 2, "tt": 3}
METRIC = "TFLOP/s & layer fwd+bwd latency, tensorized ResNet-34 convs, 1/2/4/8 B200 vs CPU"
PER_GPU_BATCH = 128
CPU_SAMPLE_BATCH = 4
WORKLOAD = "cfg2: Tucker + TT 3x3 conv layers, 256->256 ch, 14x14, fwd+bwd (all grads)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def layer_expr(kind, cr, batch):
    import paper_2401_03384_b200 as ce
    return ce.expression(ce.LayerSpec(kind, [256], [256], 3, 3, 14, 14, batch, [1] * SLOTS[kind]), cr)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and "Active" in r[3 + i]
                          and "Not" not in r[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU / reference
def cpu_reference_sample(batch_cpu=CPU_SAMPLE_BATCH, reps=1):
    """The reference's execute() (oracle/_ref: unmodified convexpr, FP64, OpenMP on all host
    cores) on a batch-`batch_cpu` sample of each layer.  Expression, ranks, plan
    (optimal, training cost mode, as the GPU arm) and the executed multiplications all come
    from the reference library.  Returns (seconds, FLOPs = 2 * multiplications, kind, cores, note)."""
    import numpy as np
    from oracle import ref
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    total_s, total_flops = 0.0, 0.0
    if ref.available():
        for k, cr in LAYERS:
            lj = json.dumps({"kind": k, "T": [256], "S": [256], "H": 3, "W": 3, "Hp": 14, "Wp": 14, "B": batch_cpu,
                             "rank": [1] * SLOTS[k]})
            expr, dims, _, _ = ref.layer(lj, cr)
            ins = [np.asarray(np.float32(ref.fill_random(d, 1000 + i)), dtype=np.float64) for i, d in enumerate(dims)]
            s, mults = ref.time_execute_mults(expr, dims, ins, "same", "training", reps=reps)
            total_s += s
            total_flops += 2.0 * mults
        return total_s, total_flops, "reference", cores, "oracle/_ref (unmodified convexpr sources)"
    # the reference could not be compiled on this host: the numpy port of it (oracle/np_oracle.py)
    from oracle import np_oracle as npo
    import paper_2401_03384_b200 as ce  # planner only (bit-exact with the reference's, tests/test_planner.py)
    for k, cr in LAYERS:
        le = layer_expr(k, cr, batch_cpu)
        p = ce.optimal(le.expr, le.dims, "same", "training")
        nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(p.to_json())["nodes"]]
        ins = [npo.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
        t0 = time.perf_counter()
        npo.execute(le.expr, le.dims, nodes, ins)
        total_s += time.perf_counter() - t0
        total_flops += 2.0 * p.flops_actual
    return total_s, total_flops, "port", 1, "oracle/np_oracle.py (numpy port; reference not built)"


def run_reference_arm(args, rank, world):
    """--impl reference: the reference's own CPU executor (forward only: it has no backward)."""
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_reference_sample(reps=1)
    secs, flops, kind, cores, src = [], None, "reference", 1, ""
    for _ in range(args.steps):
        s, flops, kind, cores, src = cpu_reference_sample(reps=1)
        secs.append(s)
    t = statistics.median(secs)
    value = flops / t / 1e12
    gpu_batch = PER_GPU_BATCH * world
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "global_batch": gpu_batch, "sample_batch": CPU_SAMPLE_BATCH,
                   "note": "the reference has no backward: its forward of the same four layers (same training-mode "
                           "plans), on a batch-%d sample; value = 2 * executed multiplications / time" % CPU_SAMPLE_BATCH},
        "projected_ms_at_global_batch": round(t * 1e3 * gpu_batch / CPU_SAMPLE_BATCH, 1),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": kind,
                         "sample": f"reference execute() forward of the 4 cfg2 layers at batch {CPU_SAMPLE_BATCH} "
                                   f"(median of {args.steps}), OMP_NUM_THREADS={cores}; {src}"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- self-launch for N > 1
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn(args):
    """`python bench.py --gpus N` outside torchrun: re-run this script under
    torch.distributed.run with N local ranks (rank 0 prints the JSON line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ----------------------------------------------------------------------------- measured TF32 peak
def measure_tf32_peak(dev):
    """Dense TF32 tensor-core peak of THIS box, for the roofline denominator only: FP32 matmul
    8192^3 with TF32 allowed (cuBLAS), best of 10, CUDA events.  Never part of the product path."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=dev)
        b = torch.randn(n, n, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        best = 1e30
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        del a, b
        return 2.0 * n ** 3 / (best * 1e-3) / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


# ----------------------------------------------------------------------------- cfg3 stack
RTR_FACT = {3: [1, 1, 3], 64: [4, 4, 4], 128: [4, 4, 8], 256: [4, 8, 8], 512: [8, 8, 8]}
RESNET34 = [(3, 64, 7, 112, 1), (64, 64, 3, 56, 6), (64, 128, 3, 28, 1), (128, 128, 3, 28, 7),
            (128, 256, 3, 14, 1), (256, 256, 3, 14, 11), (256, 512, 3, 7, 1), (512, 512, 3, 7, 5)]


def time_cfg3_stack(ctx, flush, iters=2):
    """cfg3: tensor-ring reshaped (M=3) ResNet-34 conv stack, batch 256, cr 0.1, fwd+bwd."""
    r = time_stack(ctx, flush, "rtr", 256, 0.1, iters)
    r["workload"] = "cfg3 RTR (M=3) ResNet-34 conv stack, batch 256, cr 0.1, fwd+bwd, 33 convs"
    return r


def time_cfg4_stack(ctx, flush, iters=2):
    """cfg4: CP ResNet-34 conv stack, the per-GPU shard of global batch 1024 over 8 GPUs (128),
    cr 0.1 and 1.0, fwd+bwd (one GPU: the factor-gradient all-reduce is measured by --gpus N)."""
    out = {"workload": "cfg4 CP ResNet-34 conv stack, per-GPU batch 128 (1024 / 8), fwd+bwd, 33 convs"}
    for cr in (0.1, 1.0):
        r = time_stack(ctx, flush, "cp", 128, cr, iters)
        r["images_per_s_per_gpu"] = round(128 / (r["stack_fwd_bwd_ms"] * 1e-3), 1)
        out[f"cr{cr}"] = r
    return out


def time_layer_once(ctx, flush, le, backward, iters=3):
    """Median device ms of one layer (fwd, or fwd+bwd), L2 flushed, after a warm-up."""
    import torch
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Executor
    plan = ce.optimal(le.expr, le.dims, "same", "training" if backward else "inference")
    ex = Executor(ctx, plan, backward=backward)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    dout = ctx.fill_random(plan.out_dims, 2000) if backward else None
    out = torch.empty(plan.out_dims, device=xs[0].device)
    ex.execute(xs, out)
    if backward:
        ex.backward(xs, dout)
    ts = []
    for _ in range(iters):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.torch_stream)
        ex.execute(xs, out)
        if backward:
            ex.backward(xs, dout)
        e1.record(ctx.torch_stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    fl = 2.0 * plan.flops_actual * (3.0 if backward else 1.0)
    return {"ms": round(ms, 4), "tflops": round(fl / (ms * 1e-3) / 1e12, 2)}


def time_cfg1_cfg5(ctx, flush):
    """cfg1 (CP 3x3, batch 8, 64->64, 32x32, rank 16: forward, the CPU reference's case) and
    cfg5 (CP/TK/TT/TR compression sweep at the cfg2 shape vs the dense conv through the same
    executor, fwd+bwd)."""
    import paper_2401_03384_b200 as ce
    le1 = ce.expression(ce.LayerSpec("cp", [64], [64], 3, 3, 32, 32, 8, [16]))
    cfg1 = {"workload": "cfg1 CP 3x3, B8, 64->64, 32x32, R16", "forward": time_layer_once(ctx, flush, le1, False, 10),
            "fwd_bwd": time_layer_once(ctx, flush, le1, True, 10)}
    sweep = {}
    for kind, slots in (("cp", 1), ("tk", 2), ("tt", 3), ("tr", 4)):
        for cr in (0.05, 0.1, 0.2, 0.3, 0.4, 0.5):
            le = ce.expression(ce.LayerSpec(kind, [256], [256], 3, 3, 14, 14, 128, [1] * slots), cr)
            sweep[f"{kind}_cr{cr}"] = time_layer_once(ctx, flush, le, True)
    sweep["dense"] = time_layer_once(ctx, flush,
                                     ce.expression(ce.LayerSpec("standard", [256], [256], 3, 3, 14, 14, 128, [])), True)
    return cfg1, {"workload": "cfg5 compression sweep at the cfg2 shape (B128, 256->256, 14x14), fwd+bwd, ms and "
                              "TF/s per layer; dense = bshw,tshw->bthw|hw on the same executor (no cuBLAS)",
                  "layers": sweep}


def time_stack(ctx, flush, kind, batch, cr, iters=2):
    """A ResNet-34 conv stack of `kind` layers: each distinct layer shape (stride-2 layers run
    stride-1 at output resolution) is timed (median of `iters` after a warm-up, L2 flushed)
    and weighted by its count in the 33 convs."""
    import torch
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Executor
    tot_ms, tot_fl, per = 0.0, 0.0, {}
    for s, t, k, hp, count in RESNET34:
        if kind == "rtr":
            spec = ce.LayerSpec("rtr", RTR_FACT[t], RTR_FACT[s], k, k, hp, hp, batch, [1, 1, 1, 1])
        else:
            spec = ce.LayerSpec(kind, [t], [s], k, k, hp, hp, batch, [1])
        le = ce.expression(spec, cr)
        plan = ce.optimal(le.expr, le.dims, "same", "training")
        ex = Executor(ctx, plan, backward=True)
        xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
        dout = ctx.fill_random(plan.out_dims, 2000)
        out = torch.empty(plan.out_dims, device=dout.device)
        ex.execute(xs, out)
        ex.backward(xs, dout)
        ts = []
        for _ in range(iters):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.torch_stream)
            ex.execute(xs, out)
            ex.backward(xs, dout)
            e1.record(ctx.torch_stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        fl = 6.0 * plan.flops_actual
        per[f"{s}->{t}@{hp}x{count}"] = round(ms, 3)
        tot_ms += count * ms
        tot_fl += count * fl
        del ex, xs, dout, out
        torch.cuda.empty_cache()
    return {"stack_fwd_bwd_ms": round(tot_ms, 2), "tflops": round(tot_fl / (tot_ms * 1e-3) / 1e12, 2),
            "per_layer_ms": per}


# ----------------------------------------------------------------------------- GPU arm
def time_step_math(local, flush, math, iters=3):
    """The cfg2 step (4 layers, fwd+bwd, batch 128) in another math mode of the same executor:
    "fp32" = FP32 SIMT kernels (the accuracy anchor), "3xtf32" = split operands on the tensor
    cores (~FP32 accuracy).  Eager, L2 flushed, median of `iters` after one warm-up step."""
    import torch
    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Context, Executor
    ctx = Context(local, math)
    torch.cuda.set_stream(ctx.torch_stream)
    ls, flops = [], 0.0
    for kind, cr in LAYERS:
        le = layer_expr(kind, cr, PER_GPU_BATCH)
        plan = ce.optimal(le.expr, le.dims, "same", "training")
        xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
        ls.append((Executor(ctx, plan, backward=True), xs, ctx.fill_random(plan.out_dims, 2000),
                   torch.empty(plan.out_dims, device=xs[0].device)))
        flops += 6.0 * plan.flops_actual

    def step():
        for ex, xs, dout, out in ls:
            ex.execute(xs, out)
            ex.backward(xs, dout)

    step()
    ts = []
    for _ in range(iters):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.torch_stream)
        step()
        e1.record(ctx.torch_stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    del ls
    torch.cuda.synchronize()
    return {"ms_per_step": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 2), "launch": "eager"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cfg3", action="store_true", help="skip the extra keys (cfg1, cfg3 and cfg4 stacks, cfg5 sweep)")
    ap.add_argument("--profile-json", default=None, help="write per-kernel times here")
    args = ap.parse_args()
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2401_03384_b200 as ce
    from paper_2401_03384_b200.device import Context, Executor
    from paper_2401_03384_b200.parallel import allreduce_factor_grads, allreduce_factor_grads_async

    # CE_BENCH_SHARE_GPU=1 exercises the multi-rank path of this script with more ranks than
    # GPUs (test only: NCCL refuses two ranks on one device, so the collectives go over gloo;
    # the measured path is NCCL, one GPU per rank)
    share = os.environ.get("CE_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("CE_BENCH_BACKEND", "gloo" if share else "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    ctx = Context(local, "auto")
    stream = ctx.torch_stream
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_stream(stream)  # every torch op of the bench is ordered with libce's kernels

    layers = []
    for kind, cr in LAYERS:
        le = layer_expr(kind, cr, PER_GPU_BATCH)
        plan = ce.optimal(le.expr, le.dims, "same", "training")
        ex = Executor(ctx, plan, backward=True)
        # inputs: X sharded by rank (different seeds per rank), factors identical everywhere
        xs = [ctx.fill_random(d, 1000 + i + (7919 * rank if i == 0 else 0)) for i, d in enumerate(le.dims)]
        dout = ctx.fill_random(plan.out_dims, 2000 + rank)
        fwd_flops = 2.0 * plan.flops_actual
        layers.append(dict(kind=kind, cr=cr, le=le, plan=plan, ex=ex, xs=xs, dout=dout,
                           flops=3.0 * fwd_flops, out=torch.empty(plan.out_dims, device=dev)))
    step_flops = sum(l["flops"] for l in layers)
    layer_desc = [f"{l['kind']} cr={l['cr']} R={l['le'].ranks[0]} tree={l['plan'].tree_encoding()}" for l in layers]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    def one_step():
        launches = 0
        works = []
        for l in layers:
            l["ex"].execute(l["xs"], l["out"])
            launches += l["ex"].stats.kernels_launched
            grads = l["ex"].backward(l["xs"], l["dout"])
            launches += l["ex"].stats.kernels_launched
            if world > 1:
                # factor gradients only (one bucketed NCCL all-reduce per layer, overlapping the
                # next layer's work); X gradients stay sharded
                grads, work = allreduce_factor_grads_async(grads)
                works.append(work)
            l["grads"] = grads
        for w in works:  # the step ends when every factor gradient is reduced
            if w is not None:
                w.wait()
        return launches

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    # One GPU: the whole step (4 layers, forward + backward) is captured once as a CUDA graph
    # and replayed -- how a training loop would run it; the executors launch their steps
    # straight into the capture.  (N > 1 keeps eager launches: the NCCL all-reduces.)
    # CE_BENCH_STEP_GRAPH=0: eager.
    step_graph = None
    step_launches = 0
    if world == 1 and os.environ.get("CE_BENCH_STEP_GRAPH", "1") != "0":
        step_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(step_graph, stream=stream):
            step_launches = one_step()
        step_graph.replay()
        torch.cuda.synchronize()

    times = []
    launches = 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if step_graph is not None:
                step_graph.replay()
                launches = step_launches
            else:
                launches = one_step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    ms = statistics.mean(times)
    ms_median = statistics.median(times)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * step_flops / (ms * 1e-3) / 1e12

    # per-layer fwd+bwd latency (device, median of 5 passes, events per layer)
    lat = {}
    for l in layers:
        ts = []
        for _ in range(5):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            l["ex"].execute(l["xs"], l["out"])
            l["ex"].backward(l["xs"], l["dout"])
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        lat[f"{l['kind']}_cr{l['cr']}_R{l['le'].ranks[0]}"] = round(statistics.median(ts), 4)

    # ---------------------------------------------------------------- e2e through the public API, host buffers
    pinned = []
    for l in layers:
        hin = [x.cpu().pin_memory() for x in l["xs"]]
        hd = l["dout"].cpu().pin_memory()
        hout = torch.empty(l["plan"].out_dims, pin_memory=True)
        hg = [torch.empty(x.shape, pin_memory=True) for x in l["xs"]]
        din = [torch.empty_like(x) for x in l["xs"]]
        pinned.append((hin, hd, hout, hg, din, torch.empty_like(l["dout"])))
    h2d = sum(sum(x.numel() * 4 for x in p[0]) + p[1].numel() * 4 for p in pinned)
    d2h = sum(p[2].numel() * 4 + sum(g.numel() * 4 for g in p[3]) for p in pinned)

    # PCIe is full duplex: host->device uploads run on one copy stream, device->host
    # downloads on another, both pipelined against the layers' compute on the executor
    # stream (layer i+1 uploads and layer i-1 downloads while layer i computes).
    h2d_stream, d2h_stream = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def e2e_step():
        h2d_stream.wait_stream(stream)  # previous users of the device input buffers are done
        d2h_stream.wait_stream(stream)
        up_fwd, up_bwd = [], []
        with torch.cuda.stream(h2d_stream):
            # per layer: the forward's inputs first, then dY (needed only by the backward)
            for (hin, hd, hout, hg, din, ddout) in pinned:
                for d, h in zip(din, hin):
                    d.copy_(h, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d_stream)
                up_fwd.append(ev)
                ddout.copy_(hd, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d_stream)
                up_bwd.append(ev)
        for l, (hin, hd, hout, hg, din, ddout), ef, eb in zip(layers, pinned, up_fwd, up_bwd):
            stream.wait_event(ef)
            with torch.cuda.stream(stream):
                out = l["ex"].execute(din, l["out"])
            d2h_stream.wait_stream(stream)
            with torch.cuda.stream(d2h_stream):
                hout.copy_(out, non_blocking=True)  # overlaps this layer's backward
            stream.wait_event(eb)
            with torch.cuda.stream(stream):
                grads = l["ex"].backward(din, ddout)
                if world > 1:
                    grads = allreduce_factor_grads(grads)
            d2h_stream.wait_stream(stream)
            with torch.cuda.stream(d2h_stream):
                for h, g in zip(hg, grads):
                    h.copy_(g, non_blocking=True)
                    g.record_stream(d2h_stream)
        stream.wait_stream(d2h_stream)  # the step ends when the last result is on the host

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e2e_times = []
    for _ in range(max(3, args.steps // 2)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_times.append(e0.elapsed_time(e1))
    e2e_ms = statistics.mean(e2e_times)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * step_flops / (e2e_ms * 1e-3) / 1e12

    # ---------------------------------------------------------------- live per-kernel roofline
    hbm, bf16, peak_kind = load_peaks()
    tf32_peak = measure_tf32_peak(dev)
    kern = []
    for l in layers:
        l["ex"].set_profiling(True)
        flush.fill_(1.0)
        torch.cuda.synchronize()
        l["ex"].execute(l["xs"], l["out"])
        f = l["ex"].profile(False)
        l["ex"].backward(l["xs"], l["dout"])
        b = l["ex"].profile(True)
        torch.cuda.synchronize()
        l["ex"].set_profiling(False)
        tag = f"{l['kind']}{l['cr']}"
        kern += [(tag + ":" + n, k, t, fl, by) for (n, k, t, fl, by) in f + b]
    total_k = sum(k[2] for k in kern)
    top = max(kern, key=lambda k: k[2])
    name, kind, t_ms, fl, by = top
    # DRAM traffic per launch of that kernel from the committed `ncu --set full` captures
    traffic, traffic_src = None, "profiles/ncu_traffic_r02.json"
    try:
        with open(os.path.join(ROOT, traffic_src)) as f:
            tj = json.load(f)
        if name in tj.get("kernels", {}):
            traffic = tj["kernels"][name]["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    if kind == "tc":
        ach = fl / (t_ms * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": round(tf32_peak, 1), "unit": "TFLOP/s",
                "frac": round(ach / tf32_peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                "kernel": name, "share_of_step": round(t_ms / total_k, 3),
                "peak_note": "dense TF32 measured on this box (FP32 8192^3 matmul, TF32 allowed, best of 10); "
                             f"bf16 {peak_kind} {bf16} TF/s",
                "hbm_frac": round(by / (t_ms * 1e-3) / 1e9 / hbm, 4)}
    else:
        ach = by / (t_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 4), "traffic": traffic, "traffic_source": traffic_src, "kernel": name,
                "share_of_step": round(t_ms / total_k, 3), "peak_note": f"{peak_kind} copy bandwidth"}
    # step-level attainable bound: sum over the algorithmic steps (packs excluded: they carry no
    # algorithmic work) of max(FLOPs / TF32 peak, compulsory bytes / HBM peak)
    t_att = sum(max(fl_ / (tf32_peak * 1e12), by_ / (hbm * 1e9)) for (_, k_, _, fl_, by_) in kern if k_ != "permute")
    roof["step_attainable_ms"] = round(t_att * 1e3, 4)
    roof["step_attainable_frac"] = round(t_att * 1e3 / ms, 4)
    roof["kernel_time_share"] = {k_: round(sum(t for (_, kk, t, _, _) in kern if kk == k_) / total_k, 3)
                                 for k_ in sorted({k[1] for k in kern})}
    if args.profile_json and rank == 0:
        with open(args.profile_json, "w") as f:
            json.dump([dict(name=n, kind=k, ms=t, flops=fl, bytes=by,
                            tflops=fl / (t * 1e-3) / 1e12 if t > 0 else 0, gbs=by / (t * 1e-3) / 1e9 if t > 0 else 0)
                       for (n, k, t, fl, by) in kern], f, indent=1)

    # ---------------------------------------------------------------- cfg3 stack (largest single-GPU config)
    cfg1 = cfg3 = cfg4 = cfg5 = None
    precision = None
    if rank == 0 and world == 1 and not args.no_cfg3:
        for l in layers:
            l.clear()
        torch.cuda.empty_cache()
        # the same step in the FP32 SIMT anchor and 3xTF32 modes, beside the TF32 headline
        precision = {"tf32": {"ms_per_step": round(ms, 4), "tflops": round(value, 2),
                              "launch": "graph" if step_graph is not None else "eager"},
                     "3xtf32": time_step_math(local, flush, "3xtf32"),
                     "fp32_simt": time_step_math(local, flush, "fp32")}
        torch.cuda.set_stream(stream)
        cfg3 = time_cfg3_stack(ctx, flush)
        cfg4 = time_cfg4_stack(ctx, flush)
        cfg1, cfg5 = time_cfg1_cfg5(ctx, flush)

    # ---------------------------------------------------------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s, fl_cpu, kindc, cores, src = cpu_reference_sample(CPU_SAMPLE_BATCH, reps=2)
        cpu = {"value": fl_cpu / s / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kindc,
               "sample": f"reference execute() FORWARD (no backward exists) of the 4 layers at batch "
                         f"{CPU_SAMPLE_BATCH} of 128, FP64, best of 2, {s * 1e3:.0f} ms; {src}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "ms_per_step_median": round(ms_median, 4),
            "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "tf32", "data": "synthetic (SplitMix64 fill_random, reference seeds)",
            "config": {"workload": WORKLOAD,
                       "layers": layer_desc,
                       "global_batch": PER_GPU_BATCH * world, "per_gpu_batch": PER_GPU_BATCH,
                       "parallelism": f"batch-sharded x{world}, factor-grad NCCL all-reduce" if world > 1 else "1 GPU",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "launch": "whole step replayed as one CUDA graph" if step_graph is not None
                                 else "eager (per-executor CUDA graphs)",
                       "flops_per_step_per_gpu": step_flops},
            "layer_fwd_bwd_ms": lat,
            "e2e": {"value": round(e2e_value, 3), "unit": "TFLOP/s", "ms_per_step": round(e2e_ms, 4),
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "pinned host -> H2D (copy stream) -> ce_execute + ce_backward (C-ABI) -> D2H of output "
                            "+ all grads (second copy stream), pipelined across the 4 layers"},
            "gpu_launches": launches,
            "roofline": roof,
            "cpu_baseline": cpu,
            "precision_modes": precision,
            "cfg1": cfg1,
            "cfg3_stack": cfg3,
            "cfg4_stack": cfg4,
            "cfg5_sweep": cfg5,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
