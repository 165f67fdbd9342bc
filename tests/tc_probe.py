"""Quick probe: one TC GEMM and one TC conv vs oracle (run under timeout on the GPU box)."""
import json, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_03384_b200 as ce
from paper_2401_03384_b200.device import Context, Executor, pairwise_eval
from oracle import np_oracle as npo

ctx = Context(0, "auto")
def check(expr, ld, rd, mode="same"):
    a = npo.fill_random(ld, 1).astype(np.float32); b = npo.fill_random(rd, 2).astype(np.float32)
    p = ce.optimal(expr, [ld, rd], mode)
    print(expr, ld, rd, p.describe_steps(False).splitlines()[:3], flush=True)
    out = pairwise_eval(ctx, expr, torch.tensor(a, device="cuda"), torch.tensor(b, device="cuda"), mode)
    torch.cuda.synchronize()
    op = npo.pairwise_from_expr(expr, ld, rd, mode)
    ref = npo.pairwise_eval(op, a.astype(np.float64), b.astype(np.float64))
    e = np.abs(out.cpu().numpy() - ref).max() / np.abs(ref).max()
    print("   err", e, flush=True)
    return e

check("mk,nk->mn", [128, 32], [64, 32])
check("mk,nk->mn", [256, 96], [80, 96])
check("km,kn->mn", [64, 128], [64, 64])
check("bhwr,rt->bhwt", [2, 8, 8, 36], [36, 40])
check("bshw,rs->bhwr", [2, 40, 14, 14], [24, 40])
check("bhwr,trhw->bhwt|hw", [2, 14, 14, 36], [40, 36, 3, 3])
