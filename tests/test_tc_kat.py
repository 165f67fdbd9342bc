"""Known-answer tests of the tcgen05 kind::tf32 operand layouts (GPU).

Every combination of K-major / MN-major A and B (the instruction descriptor's transpose
bits 15/16 with MN-major SWIZZLE_128B smem descriptors, LBO = 4096 B between 32-wide MN
boxes, SBO = 1024 B between 8-row K atoms) against the FP64 oracle, including ragged
M / N / K extents (TMA zero fill), a convolution whose taps shift an MN-major operand, and
the same steps with the in-smem transposer (CE_TC_NATIVE_MN=0, run in a subprocess).

Small integers make the products exact in TF32 (|x| <= 8 has <= 4 significant bits, and
sums of K <= 96 such products stay below 2^24), so these are exact-equality KATs; the
random-valued cases use the TF32 tolerance of tests/test_gpu_parity.py.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import np_oracle as npo

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (expr, left dims, right dims, expected "amn=.. bmn=.." of the TC step)
CASES = [
    ("mk,nk->mn", [128, 64], [64, 64], "amn=0 bmn=0"),
    ("km,nk->mn", [64, 128], [64, 64], "amn=1 bmn=0"),
    ("mk,kn->mn", [128, 64], [64, 64], "amn=0 bmn=1"),
    ("km,kn->mn", [64, 128], [64, 64], "amn=1 bmn=1"),
    ("km,kn->mn", [96, 256], [96, 128], "amn=1 bmn=1"),
    ("km,kn->mn", [40, 200], [40, 96], "amn=1 bmn=1"),    # ragged K (tail rows zero-filled), ragged M
    ("km,nk->mn", [72, 300], [50, 72], "amn=1 bmn=0"),    # ragged everything
    ("bshw,ts->bthw", [4, 40, 14, 16], [48, 40], "amn=1 bmn=0"),  # NCHW X: (h,w) merged M unit
    ("bshw,ths->bthw|h", [4, 40, 14, 16], [48, 3, 40], "amn=1 bmn=0"),  # taps shift the MN-major A
]


def _eval(ctx, expr, ld, rd, a, b):
    from paper_2401_03384_b200.device import pairwise_eval
    out = pairwise_eval(ctx, expr, torch.tensor(a, dtype=torch.float32, device="cuda").reshape(ld),
                        torch.tensor(b, dtype=torch.float32, device="cuda").reshape(rd))
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


def _steps(expr, ld, rd):
    import paper_2401_03384_b200 as ce
    return ce.optimal(expr, [ld, rd], "same").describe_steps(False)


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}_{c[1]}_{c[2]}" for c in CASES])
def test_operand_major_kat_exact(ctx, case):
    expr, ld, rd, majors = case
    steps = _steps(expr, ld, rd)
    assert " tc " in steps and majors in steps, steps
    rng = np.random.default_rng(5)
    a = rng.integers(-8, 9, ld).astype(np.float64)
    b = rng.integers(-8, 9, rd).astype(np.float64)
    out = _eval(ctx, expr, ld, rd, a, b)
    ref = npo.pairwise_eval(npo.pairwise_from_expr(expr, ld, rd), a, b)
    assert np.array_equal(out, ref), float(np.abs(out - ref).max())


def test_identity_selects_rows(ctx):
    """A = identity (MN-major, K = M): C = B^T exactly, so every MN box / K atom lands where
    the descriptor says (a swapped LBO/SBO permutes rows)."""
    m = 128
    a = np.eye(m)
    b = np.arange(m * 96, dtype=np.float64).reshape(m, 96) % 97 - 48
    out = _eval(ctx, "km,kn->mn", [m, m], [m, 96], a, b)
    assert np.array_equal(out, b)


def test_mn_major_conv_random(ctx):
    """Convolution with shifted taps on an MN-major operand (X in NCHW order, channels = K)."""
    expr, ld, rd = "bshw,ths->bthw|h", [4, 40, 14, 16], [48, 3, 40]
    assert "amn=1" in _steps(expr, ld, rd)
    rng = np.random.default_rng(9)
    a = rng.uniform(-1, 1, ld).astype(np.float32).astype(np.float64)
    b = rng.uniform(-1, 1, rd).astype(np.float32).astype(np.float64)
    out = _eval(ctx, expr, ld, rd, a, b)
    ref = npo.pairwise_eval(npo.pairwise_from_expr(expr, ld, rd), a, b)
    assert np.abs(out - ref).max() / np.abs(ref).max() <= 5e-3


_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2401_03384_b200.device import Context, pairwise_eval
ctx = Context(0, "auto")
rng = np.random.default_rng(5)
res = {}
for i, (expr, ld, rd) in enumerate([("km,kn->mn", [96, 256], [96, 128]), ("km,nk->mn", [72, 300], [50, 72]),
                                    ("bshw,ths->bthw|h", [4, 40, 14, 16], [48, 3, 40])]):
    a = rng.integers(-8, 9, ld).astype(np.float32); b = rng.integers(-8, 9, rd).astype(np.float32)
    out = pairwise_eval(ctx, expr, torch.tensor(a, device="cuda"), torch.tensor(b, device="cuda"))
    torch.cuda.synchronize()
    res[f"c{i}"] = out.cpu().numpy()
np.savez(sys.argv[2], **res)
"""


def test_native_and_transposer_paths_agree(tmp_path):
    """The native MN-major MMA and the in-smem transposer (CE_TC_NATIVE_MN=0) give the same
    exact integer results."""
    outs = {}
    for flag in ("1", "0"):
        f = tmp_path / f"n{flag}.npz"
        r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, str(f)], env=dict(os.environ, CE_TC_NATIVE_MN=flag),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[flag] = np.load(f)
    for k in outs["1"].files:
        assert np.array_equal(outs["1"][k], outs["0"][k]), k
