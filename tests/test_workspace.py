"""Liveness-based workspace reuse: the executor's arena holds a buffer only
from its first to its last step (the reference keeps every intermediate alive,
sequencer.cpp:421-433).  Host-only: the step list and arena sizes come from the plan
compiler, no device needed.  Correctness of the shared arena on the device is covered by
every -m gpu parity test (they run with reuse on, the default)."""
import pytest

import paper_2401_03384_b200 as ce


def _ws(kind, tf, sf, k, hp, batch, cr):
    slots = {"cp": 1, "tk": 2, "tt": 3, "tr": 4, "rtr": 4}[kind]
    le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, batch, [1] * slots), cr)
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    lines = plan.describe_steps(True, "auto").splitlines()
    vals = {l.split()[0]: int(l.split()[1]) for l in lines if l.startswith("workspace_bytes")}
    return vals["workspace_bytes"], vals["workspace_bytes_unshared"]


@pytest.mark.parametrize("case,frac", [
    # above CE_WS_TIGHT_GB (16 GB unshared): buffers share across the whole step timeline
    (("rtr", [4, 4, 8], [4, 4, 4], 3, 28, 256, 0.1), 0.6),   # cfg3 64->128 @28, B=256: 37.5 -> 20.6 GB
    # below it: sharing only along the passes' happens-before order (no new synchronisation);
    # the repack reuse and hoisting already removed most short-lived buffers of the smaller
    # layers (cfg2 TT cr1.0: 223 -> 170 MB unshared), and the row GEMMs removed conv1's
    # temporaries, so the 512-channel @7 layer is the one that still shares a lot
    (("rtr", [8, 8, 8], [4, 8, 8], 3, 7, 256, 0.1), 0.8),  # cfg3 256->512 @7: 126 -> 90 MB
])
def test_workspace_shrinks_by_liveness(case, frac):
    shared, unshared = _ws(*case)
    assert 0 < shared <= frac * unshared, (case, shared, unshared)


def test_workspace_never_exceeds_bump_layout():
    for case in [("cp", [64], [64], 3, 32, 8, None), ("tk", [256], [256], 3, 14, 128, 0.1),
                 ("tr", [256], [256], 3, 14, 128, 0.5)]:
        kind, tf, sf, k, hp, b, cr = case
        if cr is None:
            le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, b, [16]))
        else:
            le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, b, [1] * {"cp": 1, "tk": 2, "tr": 4}[kind]), cr)
        plan = ce.optimal(le.expr, le.dims, "same", "training")
        lines = plan.describe_steps(True, "auto").splitlines()
        vals = {l.split()[0]: int(l.split()[1]) for l in lines if l.startswith("workspace_bytes")}
        assert vals["workspace_bytes"] <= vals["workspace_bytes_unshared"]


def _ws2(kind, tf, sf, k, hp, batch, cr, recompute):
    slots = {"cp": 1, "tk": 2, "tt": 3, "tr": 4, "rtr": 4}[kind]
    le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, batch, [1] * slots), cr)
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    return plan.describe_steps(True, "auto", recompute=recompute)


def test_recompute_steps():
    """Gradient checkpointing: the backward pass starts with the forward
    steps that write workspace (not the root node, which writes the caller's output), into
    fresh buffers; a fused forward stencil pair no longer stores its intermediate."""
    keep = _ws2("cp", [64], [64], 3, 56, 8, 0.1, False).splitlines()
    rec = _ws2("cp", [64], [64], 3, 56, 8, 0.1, True).splitlines()
    fwd_keep = [l for l in keep if l.startswith("fwd")]
    fwd_rec = [l for l in rec if l.startswith("fwd")]
    assert len(fwd_keep) == len(fwd_rec)
    assert any("store_mid=1" in l for l in fwd_keep) and all("store_mid=1" not in l for l in fwd_rec)
    recomputed = [l for l in rec if l.startswith("bwd recompute:")]
    assert len(recomputed) == len(fwd_rec) - 1  # every forward step but the root node


def _steps(kind, tf, sf, k, hp, batch, cr):
    slots = {"cp": 1, "tk": 2, "tt": 3, "tr": 4, "rtr": 4}[kind]
    le = ce.expression(ce.LayerSpec(kind, tf, sf, k, k, hp, hp, batch, [1] * slots), cr)
    plan = ce.optimal(le.expr, le.dims, "same", "training")
    return plan.describe_steps(True, "auto")


def test_layout_hoisting_removes_intermediate_repacks():
    """cfg3 64->128 @28 (B=256): node1's 5-GB result N1 is written by its producer in the
    layout its consumer (node3) would repack it into, so node3 and the filter gradient that
    re-read it run without a repack; N0's packed layout (a 4-wide innermost axis) is not
    hoisted (its producer's stores would fragment)."""
    steps = _steps("rtr", [4, 4, 8], [4, 4, 4], 3, 28, 256, 0.1)
    assert "node3:packA" not in steps and "grad:7:packA" not in steps, steps
    assert "node1:packA" in steps
    # below the 64-MB threshold nothing is hoisted (small packs are cheap)
    assert "node3:packA" in _steps("rtr", [4, 4, 8], [4, 4, 4], 3, 28, 1, 0.1)


def test_both_operand_repack_merges_shared_k():
    """RTR 64->64 @56: X (channels-first) against the contracted kernel [t1 s1 t2 s2 t3 s3 h w]
    -- neither operand K-major -- is repacked with s1 s2 s3 innermost in both, one 64-wide K
    unit (18 K stages over the 9 taps) instead of a 4-wide unit padded to 32 (144)."""
    steps = _steps("rtr", [4, 4, 4], [4, 4, 4], 3, 56, 256, 0.1)
    node3 = [l for l in steps.splitlines() if l.startswith("fwd node3 tc")][0]
    assert " kit=18 " in node3, node3


def test_backward_reuses_large_forward_repack():
    """cfg3 64->128 @28 (B=256): dW1 = sum N0 * dN1 reads N0 in the layout node1's forward
    repack already wrote (5 GB) instead of repacking N0 again for the backward."""
    steps = _steps("rtr", [4, 4, 8], [4, 4, 4], 3, 28, 256, 0.1)
    assert "node1:packA" in steps
    assert "grad:1:packA" not in steps, steps
