"""Host planner parity: libce's parse/plan/cost/layers vs the reference, bit-exact.

Golden vectors (tests/golden/*.json) come from the compiled reference
(tests/golden/gen_golden.py); the `ref` fixture additionally cross-checks live
against oracle/_ref when it is built (build container).
"""
import json
import os

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from tests.spec_gen import random_spec

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


PLANNER = load("planner.json")
LAYERS = load("layers.json")


@pytest.mark.parametrize("chunk", range(6))
def test_random_specs_bit_exact(chunk):
    """SPEC.md:563 generator: plan JSON, tree encoding and u128 costs byte-equal to the reference."""
    for case in PLANNER[chunk * 100:(chunk + 1) * 100]:
        for row in case["plans"]:
            mk = ce.optimal if row["which"] == "optimal" else ce.left_to_right
            p = mk(case["expr"], case["dims"], case["mode"], row["cost_mode"])
            assert p.to_json() == row["json"], (case["expr"], row)
            enc = p.tree_encoding()
            assert enc == row["enc"]
            assert p.inference_cost == row["ci"] and p.training_cost == row["ct"]


def test_optimal_equals_enumeration_minimum():
    """optimal cost == min over enumerate_all on every random spec."""
    n = 0
    for case in PLANNER:
        if case["enum"] is None:
            continue
        p = ce.optimal(case["expr"], case["dims"], case["mode"], "inference")
        assert p.total_cost == case["enum"][1]
        n += 1
    assert n >= 200


def test_cost_capped_identical():
    for case in PLANNER[:200]:
        a = ce.optimal(case["expr"], case["dims"], case["mode"], "training")
        b = ce.optimal(case["expr"], case["dims"], case["mode"], "training", cost_capped=True)
        assert a.to_json() == b.to_json()


def test_layer_zoo_and_baseline_configs():
    for e in LAYERS["layers"]:
        lj = json.loads(e["layer"])
        spec = ce.LayerSpec.from_json(e["layer"])
        if e["cr"] > 0:
            le = ce.expression(spec, e["cr"])
        else:
            le = ce.expression(spec)
        assert le.expr == e["expr"], e["name"]
        assert le.dims == e["dims"]
        assert le.param_count == e["params"]
        assert le.ranks == e["ranks"] or lj["kind"] in ("standard", "interleaved-group", "separable-depthwise")
        for cm, key in (("inference", ""), ("training", "_train")):
            p = ce.optimal(le.expr, le.dims, "same", cm)
            assert p.to_json() == e["json" + key], (e["name"], cm)
            assert p.tree_encoding() == e["enc" + key]
            if "ltr_json" + key in e:
                assert ce.left_to_right(le.expr, le.dims, "same", cm).to_json() == e["ltr_json" + key]


def test_resnet34_cp_blocks():
    for key, rows in LAYERS["resnet34"].items():
        b, cr = key.split("_")
        mine = ce.resnet34_cp_blocks(int(b), float(cr))
        for (name, js), (mname, l) in zip(rows, mine):
            ref = ce.LayerSpec.from_json(js)
            assert name == mname and ref.ranks == l.ranks and ref.feature_h == l.feature_h


def test_theorem_plans():
    for t in LAYERS["theorem"]:
        spec = ce.LayerSpec.from_json(t["layer"])
        le = ce.expression(spec)
        m = len(spec.t_factors)
        n = len(le.dims)
        joins, cur = [], 1
        for i in range(2, m + 1):
            joins.append((cur, i))
            cur = n + len(joins) - 1
        if spec.kind == "rtk":
            joins.append((cur, m + 2))
            cur = n + len(joins) - 1
        joins.append((cur, m + 1))
        cur = n + len(joins) - 1
        joins.append((cur, 0))
        p = ce.plan_from_joins(le.expr, le.dims, joins, "same", t["cost_mode"])
        assert p.to_json() == t["json"] and p.tree_encoding() == t["enc"]


def test_spec_known_answers():
    # SPEC.md:283 / 294-295
    p = ce.optimal("abc,ade->bcde", [[2, 3, 4], [2, 5, 6]])
    assert p.total_cost == 720
    assert ce.optimal("ij,jk,kl->il", [[2, 3], [3, 4], [4, 5]]).total_cost == 64
    assert ce.plan_from_joins("ij,jk,kl->il", [[2, 3], [3, 4], [4, 5]], [(1, 2), (0, 3)]).total_cost == 90
    # SPEC.md:440, 432
    assert ce.rank_for_compression(ce.LayerSpec("cp", [64], [64], 3, 3, 32, 32, 1, [1]), 1.0) == 275
    assert ce.expression(ce.LayerSpec("rcp", [2, 2, 2], [2, 2, 2], 3, 3, 8, 8, 1, [4])).param_count == 84
    # flops_actual SPEC.md:234-236 (via the plan's executed-MAC total)
    assert ce.optimal("ij,jk->ik", [[2, 3], [3, 4]]).flops_actual == 24
    assert ce.optimal("x,x->x|x", [[2], [2]], "full").flops_actual == 4
    assert ce.optimal("ab,c->abc", [[2, 3], [4]]).flops_actual == 24


def test_parse_render_classify_and_errors():
    s = ce.parse("bsh, tsh -> bth | h")
    assert s.rendered == "bsh,tsh->bth|h"
    assert s.classes == {"b": "free", "h": "convolution", "s": "contraction", "t": "free"}
    assert ce.parse("gtsh,bgsh->bgth|h").classes["g"] == "batch"
    assert ce.parse("abc->ab").classes["c"] == "self-contraction"
    assert ce.render("b(s1)hw,r(t1)(s1)hw->b(t1)hw|h,w") == "b(s1)hw,r(t1)(s1)hw->b(t1)hw|hw"
    for bad in ("ab,bc", "a(b->a", "aa->a", "ab,bc->ad", "ab,bc->ac|a", "ab,,bc->ac", "ab->a->b", "a-b"):
        with pytest.raises(ce.ParseError):
            ce.parse(bad)
    with pytest.raises(ce.ShapeError):
        ce.optimal("ij,jk->ik", [[2, 3], [4, 5]])
    with pytest.raises(ce.ShapeError):
        ce.optimal("ij,jk->ik", [[2, 3]])


def test_live_against_reference(ref):
    """Fresh random specs (different seed than the goldens), checked live against oracle/_ref."""
    rng = np.random.default_rng(777)
    n = 0
    while n < 150:
        expr, dims, mode = random_spec(rng, 2, 6, dmax=7)
        try:
            js, enc, ci, ct = ref.plan(expr, dims, mode, "training")
        except ref.RefError as e:
            with pytest.raises(ce.CeError) as ei:
                ce.optimal(expr, dims, mode, "training")
            assert ei.value.code == e.code
            continue
        p = ce.optimal(expr, dims, mode, "training")
        assert p.to_json() == js and p.tree_encoding() == enc and p.inference_cost == ci
        n += 1


def test_parse_errors_match_reference(ref):
    assert ce.render("(a b)->(ab)") == ref.parse("(a b)->(ab)")[0] == "(ab)->(ab)"
    for bad in ("ab,bc", "a(b->a", "aa->a", "ab,bc->ad", "ab,bc->ac|a", "ab,,bc->ac", "a)->a",
                "ab,bc->ac|", "ab,bc->ac|b,", "ab->a->b", "a-b", "1a->a", "()->a"):
        with pytest.raises(ref.RefError) as r:
            ref.parse(bad)
        with pytest.raises(ce.CeError) as m:
            ce.parse(bad)
        assert m.value.code == r.value.code
        assert str(r.value).split("] ", 1)[1] in str(m.value)
