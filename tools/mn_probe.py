"""Probe: MN-major tf32 operand layouts (env knobs CE_TC_MN_*) on small exact-integer GEMMs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2401_03384_b200.device import Context, pairwise_eval
from oracle import np_oracle as npo
ctx = Context(0, "auto")
rng = np.random.default_rng(5)
res = []
for expr, ld, rd in [("km,nk->mn", [64, 128], [64, 64]), ("mk,kn->mn", [128, 64], [64, 64]),
                     ("km,kn->mn", [64, 128], [64, 64]), ("km,kn->mn", [96, 256], [96, 128])]:
    a = rng.integers(-8, 9, ld).astype(np.float32); b = rng.integers(-8, 9, rd).astype(np.float32)
    out = pairwise_eval(ctx, expr, torch.tensor(a, device="cuda"), torch.tensor(b, device="cuda")).cpu().numpy()
    ref = npo.pairwise_eval(npo.pairwise_from_expr(expr, ld, rd), a.astype(float), b.astype(float))
    err = np.abs(out - ref).max()
    # is the output a row / column permutation of ref?
    rowmatch = sum(any(np.array_equal(out[i], ref[j]) for j in range(ref.shape[0])) for i in range(out.shape[0]))
    res.append(f"{expr}{ld}{rd}: maxerr={err:.3g} |out|max={np.abs(out).max():.3g} rows_found={rowmatch}/{out.shape[0]}")
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("CE_TC_MN"))
print(tag or "default", "\n  " + "\n  ".join(res), flush=True)
