"""Kernel steps of one cfg3 RTR layer (no GPU).  usage: python tools/describe_rtr.py T S k Hp"""
import os
sys_path = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import sys
sys.path.insert(0, sys_path)
import sys, bench, paper_2401_03384_b200 as ce
T, S, k, hp = (int(x) for x in sys.argv[1:5])
le = ce.expression(ce.LayerSpec("rtr", bench.RTR_FACT[T], bench.RTR_FACT[S], k, k, hp, hp, 256, [1,1,1,1]), 0.1)
p = ce.optimal(le.expr, le.dims, "same", "training")
print(p.tree_encoding())
print(p.describe_steps(True))
