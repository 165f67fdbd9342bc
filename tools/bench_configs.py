"""Measure every BASELINE.json config on one B200 -> JSON.

  python tools/bench_configs.py [--out profiles/configs_r01.json] [--quick]

cfg1  CP 3x3, batch 8, 64->64, 32x32, rank 16: forward latency (inference plan) and
      fwd+bwd, plus the reference CPU executor on the same forward (all host cores).
cfg2  Tucker/TT 3x3, batch 128, 256->256, 14x14: fwd+bwd per layer (the bench.py workload).
cfg3  RTR (M=3) ResNet-34 conv stack at ImageNet resolution, batch 256, cr 0.1, fwd+bwd.
      stride-2 layers run as stride-1 Same at output resolution (conv_einsum has no
      stride); each distinct layer shape is timed once and weighted by its
      count in the 33-conv stack.
cfg4  CP ResNet-34 stack, per-GPU batch 128 (= global 1024 over 8 GPUs), cr 0.1 and 1.0,
      fwd+bwd (one GPU: the all-reduce is measured by bench.py --gpus N).
cfg5  CP/TK/TT/TR at cr 0.05..0.5 and the dense conv `bshw,tshw->bthw|hw` through the
      same executor, cfg2 shape, fwd+bwd.
Timing: CUDA events on the executor stream, warm-up first, L2 flushed (256 MiB write)
before each timed iteration, median of the iterations.  FLOPs = 2 x flops_actual per node
(+ the same per requested gradient), exactly as bench.py.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2401_03384_b200 as ce  # noqa: E402
from paper_2401_03384_b200.device import Context, Executor  # noqa: E402

RTR_FACT = {3: [1, 1, 3], 64: [4, 4, 4], 128: [4, 4, 8], 256: [4, 8, 8], 512: [8, 8, 8]}
# ResNet-34 convs at output resolution: (S, T, k, H', count)
RESNET34 = [(3, 64, 7, 112, 1), (64, 64, 3, 56, 6), (64, 128, 3, 28, 1), (128, 128, 3, 28, 7),
            (128, 256, 3, 14, 1), (256, 256, 3, 14, 11), (256, 512, 3, 7, 1), (512, 512, 3, 7, 5)]


def time_layer(ctx, le, backward, iters, flush):
    cost = "training" if backward else "inference"
    plan = ce.optimal(le.expr, le.dims, "same", cost)
    ex = Executor(ctx, plan, backward=backward)
    xs = [ctx.fill_random(d, 1000 + i) for i, d in enumerate(le.dims)]
    dout = ctx.fill_random(plan.out_dims, 2000) if backward else None
    out = torch.empty(plan.out_dims, device="cuda")
    st = ctx.torch_stream

    def step():
        ex.execute(xs, out)
        if backward:
            ex.backward(xs, dout)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        step()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    fl = 2.0 * plan.flops_actual * (3.0 if backward else 1.0)
    del ex, xs, dout, out
    return {"expr": le.expr, "ranks": le.ranks, "params": le.param_count, "tree": plan.tree_encoding(),
            "ms": round(ms, 4), "tflops": round(fl / (ms * 1e-3) / 1e12, 2), "flops": fl}


def cpu_forward(le, reps=3):
    """The reference executor (oracle/_ref, FP64, OpenMP all cores), forward, best of reps."""
    import numpy as np
    from oracle import ref
    if not ref.available():
        return None
    ins = [np.asarray(np.float32(ref.fill_random(d, 1000 + i)), dtype=np.float64) for i, d in enumerate(le.dims)]
    s = ref.time_execute(le.expr, le.dims, ins, "same", "inference", reps=reps)
    plan = ce.optimal(le.expr, le.dims, "same", "inference")
    return {"s": s, "tflops": 2.0 * plan.flops_actual / s / 1e12, "cores": os.cpu_count()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "configs_r01.json"))
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--quick", action="store_true", help="fewer cfg5 points")
    ap.add_argument("--only", default="cfg1,cfg2,cfg3,cfg4,cfg5", help="comma-separated subset of configs")
    args = ap.parse_args()
    only = set(args.only.split(","))
    ctx = Context(0, "auto")
    torch.cuda.set_stream(ctx.torch_stream)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")
    res = {"device": torch.cuda.get_device_name(0), "timestamp": time.time(), "l2": "flushed before each iteration"}

    # cfg1
    if "cfg1" in only:
        le = ce.expression(ce.LayerSpec("cp", [64], [64], 3, 3, 32, 32, 8, [16]))
        res["cfg1"] = {"forward": time_layer(ctx, le, False, 20, flush), "fwd_bwd": time_layer(ctx, le, True, 20, flush),
                       "cpu_reference_forward": cpu_forward(le)}
        print("cfg1", res["cfg1"]["forward"]["ms"], flush=True)

    # cfg2
    if "cfg2" in only:
        res["cfg2"] = {}
        for kind, cr in [("tk", 0.1), ("tk", 0.25), ("tk", 1.0), ("tt", 0.1), ("tt", 0.25), ("tt", 1.0)]:
            slots = {"tk": 2, "tt": 3}[kind]
            le = ce.expression(ce.LayerSpec(kind, [256], [256], 3, 3, 14, 14, 128, [1] * slots), cr)
            res["cfg2"][f"{kind}_cr{cr}"] = time_layer(ctx, le, True, args.iters, flush)
            print("cfg2", kind, cr, res["cfg2"][f"{kind}_cr{cr}"]["ms"], flush=True)

    # cfg3: RTR stack, batch 256, cr 0.1
    if "cfg3" in only:
        layers, tot_ms, tot_fl = [], 0.0, 0.0
        for s, t, k, hp, count in RESNET34:
            le = ce.expression(ce.LayerSpec("rtr", RTR_FACT[t], RTR_FACT[s], k, k, hp, hp, 256, [1, 1, 1, 1]), 0.1)
            r = time_layer(ctx, le, True, args.iters, flush)
            r.update({"S": s, "T": t, "k": k, "Hp": hp, "count": count})
            layers.append(r)
            tot_ms += count * r["ms"]
            tot_fl += count * r["flops"]
            print("cfg3", s, t, hp, r["ms"], flush=True)
            torch.cuda.empty_cache()
        res["cfg3"] = {"batch": 256, "cr": 0.1, "layers": layers, "stack_fwd_bwd_ms": round(tot_ms, 3),
                       "stack_tflops": round(tot_fl / (tot_ms * 1e-3) / 1e12, 2)}

    # cfg4: CP stack, per-GPU batch 128
    if "cfg4" in only:
        res["cfg4"] = {}
        for cr in (0.1, 1.0):
            layers, tot_ms, tot_fl = [], 0.0, 0.0
            for s, t, k, hp, count in RESNET34:
                le = ce.expression(ce.LayerSpec("cp", [t], [s], k, k, hp, hp, 128, [1]), cr)
                r = time_layer(ctx, le, True, args.iters, flush)
                r.update({"S": s, "T": t, "k": k, "Hp": hp, "count": count})
                layers.append(r)
                tot_ms += count * r["ms"]
                tot_fl += count * r["flops"]
                torch.cuda.empty_cache()
            res["cfg4"][f"cr{cr}"] = {"per_gpu_batch": 128, "layers": layers, "stack_fwd_bwd_ms": round(tot_ms, 3),
                                      "stack_tflops": round(tot_fl / (tot_ms * 1e-3) / 1e12, 2),
                                      "images_per_s_per_gpu": round(128 / (tot_ms * 1e-3), 1)}
            print("cfg4", cr, tot_ms, flush=True)

    # cfg5: compression sweep + dense
    if "cfg5" in only:
        crs = [0.05, 0.1, 0.5] if args.quick else [0.05, 0.1, 0.2, 0.3, 0.4, 0.5]
        sweep = {}
        for kind in ("cp", "tk", "tt", "tr"):
            slots = {"cp": 1, "tk": 2, "tt": 3, "tr": 4}[kind]
            for cr in crs:
                le = ce.expression(ce.LayerSpec(kind, [256], [256], 3, 3, 14, 14, 128, [1] * slots), cr)
                sweep[f"{kind}_cr{cr}"] = time_layer(ctx, le, True, args.iters, flush)
        le = ce.expression(ce.LayerSpec("standard", [256], [256], 3, 3, 14, 14, 128, []))
        sweep["dense"] = time_layer(ctx, le, True, args.iters, flush)
        res["cfg5"] = sweep
        print("cfg5 dense", sweep["dense"]["ms"], flush=True)

    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
