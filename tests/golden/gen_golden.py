"""Generates the committed golden vectors from the COMPILED REFERENCE.

Run in the build container (needs /root/reference and `make -C oracle`):
    python tests/golden/gen_golden.py
Outputs (small JSON, committed): planner.json, pairwise.json, execute.json, layers.json.
Inputs are regenerated from SplitMix64 seeds (reference fill_random, tensor.cpp:125-130),
so fixtures store only seeds + reference outputs.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import ref  # noqa: E402
from spec_gen import random_spec  # noqa: E402

LAYER_KINDS = ["standard", "cp", "rcp", "tk", "rtk", "tt", "rtt", "tr", "rtr", "bt", "ht",
               "interleaved-group", "separable-depthwise"]


def layer_json(kind, T, S, H=3, W=3, Hp=8, Wp=8, B=2, rank=None):
    d = {"kind": kind, "T": T, "S": S, "H": H, "W": W, "Hp": Hp, "Wp": Wp, "B": B}
    if rank is not None:
        d["rank"] = rank
    return json.dumps(d)


def toy_layers():
    """All 13 kinds at toy dims (dims <= 4, H'=W'=8)."""
    out = []
    for kind in LAYER_KINDS:
        if kind in ("rcp", "rtk", "rtt", "rtr", "bt"):
            T, S = [2, 2, 2], [2, 2, 2]
        elif kind == "ht":
            T, S = [2, 2, 2], [2, 2, 2]
        elif kind == "interleaved-group":
            T, S = [2, 2], [2, 2]
        else:
            T, S = [4], [4]
        slots = {"standard": 0, "interleaved-group": 0, "separable-depthwise": 0, "cp": 1, "rcp": 1, "tk": 2,
                 "rtk": 4, "tt": 3, "rtt": 3, "tr": 4, "rtr": 4, "bt": 5, "ht": 6}[kind]
        rank = [3] * slots if slots > 1 else (3 if slots == 1 else None)
        Hp = Wp = 8
        if kind == "interleaved-group":
            Hp = Wp = 3  # h,w are 3-way -> circular with equal dims (tensor.cpp:217-218)
        out.append((kind, layer_json(kind, T, S, Hp=Hp, Wp=Wp, rank=rank)))
    return out


BASELINE_LAYERS = [
    ("cfg1 CP B8 64->64 32x32 R16", layer_json("cp", [64], [64], Hp=32, Wp=32, B=8, rank=16), 0.0),
    ("cfg2 TK cr0.1", layer_json("tk", [256], [256], Hp=14, Wp=14, B=128, rank=1), 0.1),
    ("cfg2 TK cr0.25", layer_json("tk", [256], [256], Hp=14, Wp=14, B=128, rank=1), 0.25),
    ("cfg2 TK cr1.0", layer_json("tk", [256], [256], Hp=14, Wp=14, B=128, rank=1), 1.0),
    ("cfg2 TT cr0.1", layer_json("tt", [256], [256], Hp=14, Wp=14, B=128, rank=1), 0.1),
    ("cfg2 TT cr0.5", layer_json("tt", [256], [256], Hp=14, Wp=14, B=128, rank=1), 0.5),
    ("cfg2 TT cr1.0", layer_json("tt", [256], [256], Hp=14, Wp=14, B=128, rank=1), 1.0),
    ("cfg2 TR cr0.1", layer_json("tr", [256], [256], Hp=14, Wp=14, B=128, rank=1), 0.1),
    ("cfg3 RTR conv2_x cr0.1", layer_json("rtr", [4, 4, 4], [4, 4, 4], Hp=56, Wp=56, B=256, rank=1), 0.1),
    ("cfg3 RTR conv5_x cr1.0", layer_json("rtr", [8, 8, 8], [8, 8, 8], Hp=7, Wp=7, B=256, rank=1), 1.0),
    ("dense cfg2 shape", layer_json("standard", [256], [256], Hp=14, Wp=14, B=128), 0.0),
]


def main():
    rng = np.random.default_rng(12345)
    # ---------------------------------------------------------------- planner
    planner = []
    while len(planner) < 600:
        expr, dims, mode = random_spec(rng)
        try:
            rows = []
            for cm in ("inference", "training"):
                for which in ("optimal", "ltr"):
                    js, enc, ci, ct = ref.plan(expr, dims, mode, cm, which)
                    rows.append({"cost_mode": cm, "which": which, "json": js, "enc": enc, "ci": ci, "ct": ct})
            n = len(dims)
            enum = ref.enumerate_min(expr, dims, mode, "inference") if n <= 5 else None
        except ref.RefError:
            continue
        planner.append({"expr": expr, "dims": dims, "mode": mode, "plans": rows, "enum": enum})
    layers = []
    for name, lj in toy_layers():
        e, d, pc, rk = ref.layer(lj)
        entry = {"name": name, "layer": lj, "cr": 0.0, "expr": e, "dims": d, "params": pc, "ranks": rk}
        js, enc, ci, ct = ref.plan(e, d, "same", "inference", "optimal")
        entry.update({"json": js, "enc": enc})
        jt, et, _, _ = ref.plan(e, d, "same", "training", "optimal")
        entry.update({"json_train": jt, "enc_train": et})
        layers.append(entry)
    for name, lj, cr in BASELINE_LAYERS:
        e, d, pc, rk = ref.layer(lj, cr)
        entry = {"name": name, "layer": lj, "cr": cr, "expr": e, "dims": d, "params": pc, "ranks": rk}
        for cm, key in (("inference", ""), ("training", "_train")):
            js, enc, ci, ct = ref.plan(e, d, "same", cm, "optimal")
            entry.update({"json" + key: js, "enc" + key: enc})
            jl, el, _, _ = ref.plan(e, d, "same", cm, "ltr")
            entry.update({"ltr_json" + key: jl})
        layers.append(entry)
    resnet = {f"{b}_{cr}": ref.resnet34(b, cr) for b in (1, 128, 1024) for cr in (0.1, 1.0)}
    theorem = []
    for lj in (layer_json("rcp", [2, 2, 2], [2, 2, 2], Hp=32, Wp=32, B=2, rank=8),
               layer_json("rtk", [2, 2, 2], [2, 2, 2], Hp=16, Wp=16, B=2, rank=[4, 2, 2, 2])):
        for cm in ("inference", "training"):
            js, enc = ref.theorem_plan(lj, cm)
            theorem.append({"layer": lj, "cost_mode": cm, "json": js, "enc": enc})

    # ---------------------------------------------------------------- pairwise
    pairwise = []
    # SPEC.md:221-225 / SURVEY Appendix A.1 known answers with explicit data
    kats = [("x,x->x|x", [3], [3], "circular", [1, 0, 0], [1, 2, 3]),
            ("x,x->x|x", [2], [2], "full", [1, 1], [1, 1]),
            ("x,x->x|x", [5], [3], "same", [1, 2, 3, 4, 5], [1, 0, 0]),
            ("x,x->x|x", [5], [2], "same", [1, 2, 3, 4, 5], [1, 10]),
            ("x,x->x|x", [5], [3], "valid", [1, 2, 3, 4, 5], [1, 0, 0]),
            ("x,x->x|x", [5], [3], "full", [1, 2, 3, 4, 5], [1, 0, 0]),
            ("x,x->x|x", [3], [5], "same", [1, 0, 0], [1, 2, 3, 4, 5]),
            ("ij,jk->ik", [2, 2], [2, 2], "same", [1, 2, 3, 4], [1, 0, 0, 1]),
            ("x,y->xy", [2], [2], "same", [1, 2], [3, 4])]
    for expr, ld, rd, mode, a, b in kats:
        fa, costs, rdims, res = ref.pairwise(expr, [ld, rd], np.array(a, float), np.array(b, float), mode)
        pairwise.append({"expr": expr, "ldims": ld, "rdims": rd, "mode": mode, "a": a, "b": b, "flops": fa,
                         "costs": list(costs), "rdims_out": rdims, "out": res.ravel().tolist()})
    seed = 100
    while len(pairwise) < 260:
        expr, dims, mode = random_spec(rng, 2, 2, dmax=5)
        try:
            fa, costs, rdims, _ = ref.pairwise(expr, dims, None, None, mode)
        except ref.RefError:
            continue
        if int(np.prod(rdims or [1])) > 400:
            continue
        a = ref.fill_random(dims[0], seed)
        b = ref.fill_random(dims[1], seed + 1)
        _, _, _, res = ref.pairwise(expr, dims, a, b, mode)
        pairwise.append({"expr": expr, "ldims": dims[0], "rdims": dims[1], "mode": mode, "seeds": [seed, seed + 1],
                         "flops": fa, "costs": list(costs), "rdims_out": rdims, "out": res.ravel().tolist()})
        seed += 2

    # ---------------------------------------------------------------- execute
    execute = []
    while len(execute) < 60:
        expr, dims, mode = random_spec(rng, 1, 5, dmax=4)
        try:
            js, enc, _, _ = ref.plan(expr, dims, mode)
        except ref.RefError:
            continue
        nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(js)["nodes"]]
        seeds = [1000 + i for i in range(len(dims))]
        ins = [ref.fill_random(d, s) for d, s in zip(dims, seeds)]
        from oracle import np_oracle as npo
        shape = list(npo.execute(expr, dims, nodes, ins, mode)[0].shape)
        if int(np.prod(shape or [1])) > 600:
            continue
        out, mults, peak, _ = ref.execute(expr, dims, ins, shape, mode)
        execute.append({"expr": expr, "dims": dims, "mode": mode, "seeds": seeds, "shape": shape,
                        "out": out.ravel().tolist(), "mults": mults, "peak": peak})
    for name, lj in toy_layers():
        e, d, pc, rk = ref.layer(lj)
        if max(len(x) for x in d) > 8:
            continue
        js, _, _, _ = ref.plan(e, d)
        nodes = [(n["left"], n["right"], n["result"]) for n in json.loads(js)["nodes"]]
        seeds = [1000 + i for i in range(len(d))]
        ins = [ref.fill_random(x, s) for x, s in zip(d, seeds)]
        from oracle import np_oracle as npo
        shape = list(npo.execute(e, d, nodes, ins)[0].shape)
        out, mults, peak, _ = ref.execute(e, d, ins, shape)
        execute.append({"expr": e, "dims": d, "mode": "same", "seeds": seeds, "shape": shape, "layer": name,
                        "out": out.ravel().tolist(), "mults": mults, "peak": peak})

    def dump(name, obj):
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(obj, f, separators=(",", ":"))

    dump("planner.json", planner)
    dump("layers.json", {"layers": layers, "resnet34": resnet, "theorem": theorem})
    dump("pairwise.json", pairwise)
    dump("execute.json", execute)
    print(len(planner), len(layers), len(pairwise), len(execute))


if __name__ == "__main__":
    main()
