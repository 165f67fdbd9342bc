"""The reference-side binding (include/ce/convexpr_shim.hpp) compiled against
the unmodified reference headers and objects, replaying reference-built plans through libce.

CPU: the shim compiles and links (oracle/Makefile `shim` target -> oracle/_ref/shim_check),
where /root/reference exists.  GPU: oracle/_ref/shim_check runs optimal, left_to_right,
from_joins, hand-edited and mixed-mode (full / valid / circular) plans through both the
reference's execute() and convexpr_b200::execute(); the output shape, ExecutionResult
.multiplications and .peak_intermediate_elements must be identical and the output within
the FP32 (1e-5) / TF32 (5e-3) tolerance.
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_check")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/src"), reason="reference sources absent")
def test_shim_compiles_against_reference():
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "shim"], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert os.access(BIN, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("math,tol", [("fp32", 1e-5), ("auto", 5e-3)])
def test_shim_replays_reference_plans(math, tol):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.access(BIN, os.X_OK):
        pytest.skip("oracle/_ref/shim_check not built (build() builds it where /root/reference exists)")
    r = subprocess.run([BIN, "--math", math], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(rows) >= 12, r.stdout
    names = {row["case"] for row in rows}
    for must in ("cp left_to_right same", "cp from_joins full", "cp optimal mixed h=full w=circular",
                 "cp hand-edited result order", "three-way circular"):
        assert must in names
    for row in rows:
        assert row["shape_equal"] and row["mults_equal"] and row["peak_equal"], row
        assert row["err"] <= tol, row
