"""Kernel steps (fwd + bwd) of every BASELINE layer the bench times, for diffing planner
changes without a GPU.  usage: python tools/describe_all.py > steps.txt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2401_03384_b200 as ce  # noqa: E402


def show(name, le):
    p = ce.optimal(le.expr, le.dims, "same", "training")
    print(f"## {name} {p.tree_encoding()}")
    print(p.describe_steps(True))


for kind, cr in bench.LAYERS:
    show(f"cfg2 {kind} {cr}", bench.layer_expr(kind, cr, 128))
for s, t, k, hp, count in bench.RESNET34:
    show(f"cfg3 {s}->{t}@{hp}", ce.expression(ce.LayerSpec("rtr", bench.RTR_FACT[t], bench.RTR_FACT[s], k, k, hp, hp, 256,
                                                           [1, 1, 1, 1]), 0.1))
    for cr in (0.1, 1.0):
        show(f"cfg4 {s}->{t}@{hp} cr{cr}", ce.expression(ce.LayerSpec("cp", [t], [s], k, k, hp, hp, 128, [1]), cr))
for kind, slots in (("cp", 1), ("tk", 2), ("tt", 3), ("tr", 4)):
    for cr in (0.05, 0.1, 0.2, 0.3, 0.4, 0.5):
        show(f"cfg5 {kind} {cr}", ce.expression(ce.LayerSpec(kind, [256], [256], 3, 3, 14, 14, 128, [1] * slots), cr))
