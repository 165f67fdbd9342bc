import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2401_03384_b200.device import Context, pairwise_eval
from oracle import np_oracle as npo
ctx = Context(0, "auto")
for expr, ld, rd in [("km,kn->mn", [32, 128], [32, 64]), ("mk,kn->mn", [128, 32], [32, 64])]:
    a = npo.fill_random(ld, 1).astype(np.float32); b = npo.fill_random(rd, 2).astype(np.float32)
    out = pairwise_eval(ctx, expr, torch.tensor(a, device="cuda"), torch.tensor(b, device="cuda")).cpu().numpy()
    op = npo.pairwise_from_expr(expr, ld, rd); ref = npo.pairwise_eval(op, a.astype(float), b.astype(float))
    print(os.environ.get("TAG"), expr, "max|y|=%.3g max|ref|=%.3g err=%.3g" % (np.abs(out).max(), np.abs(ref).max(), np.abs(out-ref).max()/np.abs(ref).max()), "y[0,:4]", out[0,:4], "ref[0,:4]", ref[0,:4])
