"""The SPEC command-line interface -- ce_cli over the C-ABI.

Host-only tests cover analyze / layer / bench and every documented exit code (0 ok,
2 parse, 3 shape, 1 other); eval (the device executor) is -m gpu, including
its 4 numerical-mismatch code and the tensor wire formats it writes.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from paper_2401_03384_b200 import wire

CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2401_03384_b200", "ce_cli")


def run(*args):
    p = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=120)
    return p.returncode, p.stdout, p.stderr


def test_cli_built():
    assert os.access(CLI, os.X_OK), "make -C paper_2401_03384_b200/csrc builds ce_cli"


def test_analyze_example_and_json_round_trip():
    # ij,jk,kl->il -> optimal 64, naive 64, speedup 1.0
    rc, out, _ = run("analyze", "--expr", "ij,jk,kl->il", "--shapes", '{"dims":[[2,3],[3,4],[4,5]]}', "--json")
    assert rc == 0
    j = json.loads(out)
    assert j["optimal"]["inference_cost"] == "64" and j["left_to_right"]["inference_cost"] == "64"
    assert j["speedup"]["inference"] == 1.0
    # the embedded plan JSON is the planner's plan_to_json (byte-equal to the reference's)
    plan = ce.optimal("ij,jk,kl->il", [[2, 3], [3, 4], [4, 5]])
    assert json.dumps(j["optimal"]["plan"], separators=(",", ":"), sort_keys=True) == plan.to_json()


def test_analyze_layer_descriptor_speedup():
    # RCP M=3 descriptor -> speedup > 1 (Theorem 1)
    desc = '{"kind":"RCP","T":[4,4,4],"S":[4,4,4],"H":3,"W":3,"Hp":32,"Wp":32,"B":8,"rank":8}'
    rc, out, _ = run("analyze", "--layer", desc, "--cr", "0.5", "--json")
    assert rc == 0
    j = json.loads(out)
    assert j["speedup"]["inference"] >= 1.0
    rc, out, _ = run("analyze", "--layer", desc)
    assert rc == 0 and "speedup" in out


@pytest.mark.parametrize("args,code", [
    (("analyze", "--expr", "ij,,jk->ik", "--shapes", "[[2,3],[3,4]]"), 2),         # parse error
    (("analyze", "--expr", "ij,jk->ik", "--shapes", "[[2,3],[4,4]]"), 3),          # unequal dims
    (("analyze", "--expr", "ij,jk->ik", "--shapes", "[[2,3]]"), 3),                # wrong input count
    (("bench", "--suite", "nope"), 1),                                            # unknown suite
    (("layer", "--kind", "nope", "--desc", '{"T":[4],"S":[4],"H":3,"W":3,"Hp":8,"Wp":8}'), 1),
    (("frobnicate",), 1),
    (("analyze", "--expr"), 1),
])
def test_exit_codes(args, code):
    rc, _, err = run(*args)
    assert rc == code, err
    assert err.strip()  # diagnostics go to stderr


def test_layer_examples():
    # SPEC.md:522-526
    rc, out, _ = run("layer", "--kind", "standard", "--desc", '{"T":[4],"S":[4],"H":3,"W":3,"Hp":8,"Wp":8,"B":1}')
    assert rc == 0 and "bshw,tshw->bthw|hw" in out
    rc, out, _ = run("layer", "--kind", "cp", "--desc", '{"T":[64],"S":[64],"H":3,"W":3,"Hp":32,"Wp":32,"B":8}',
                     "--cr", "1.0", "--json")
    assert rc == 0 and json.loads(out)["ranks"] == [275]
    rc, out, _ = run("layer", "--kind", "ht", "--desc", '{"T":[2,2,2],"S":[2,2,2],"H":3,"W":3,"Hp":8,"Wp":8}')
    assert rc == 0 and "(r4)(r5)" in out


def test_bench_resnet34_cp():
    # every row optimal < left-to-right, speedups increasing conv3_x -> conv5_x,
    # and the speedup column independent of the batch
    rc, out, _ = run("bench", "--suite", "resnet34-cp", "--batch", "128", "--cr", "1.0", "--json")
    assert rc == 0
    rows = json.loads(out)
    assert [r["layer"] for r in rows] == ["conv1", "conv2_x", "conv3_x", "conv4_x", "conv5_x"]
    assert all(int(r["optimal"]) < int(r["left_to_right"]) for r in rows)
    sp = [r["speedup"] for r in rows]
    assert sp[2] < sp[3] < sp[4]
    rc, out1, _ = run("bench", "--suite", "resnet34-cp", "--batch", "1", "--cr", "1.0", "--json")
    assert [r["speedup"] for r in json.loads(out1)] == sp


@pytest.mark.gpu
def test_eval_both_plans_and_outputs(tmp_path):
    # "bsh,tsh->bth|h" --plan both -> deviation within tolerance, exit 0
    rc, out, err = run("eval", "--expr", "bsh,tsh->bth|h", "--shapes", "[[2,3,9],[4,3,3]]", "--seed", "1",
                       "--plan", "both")
    assert rc == 0, err
    assert "max relative deviation" in out
    # CP layer (two conv atoms shared by 2 inputs each) through both plans in FP32
    desc = '{"kind":"CP","T":[8],"S":[6],"H":3,"W":3,"Hp":10,"Wp":10,"B":2,"rank":5}'
    rc, out, err = run("eval", "--layer", desc, "--seed", "3", "--plan", "both")
    assert rc == 0, err
    # --out in both wire formats, read back with the reference's formats
    js, bn = str(tmp_path / "y.json"), str(tmp_path / "y.bin")
    assert run("eval", "--expr", "bsh,tsh->bth|h", "--shapes", "[[2,3,9],[4,3,3]]", "--seed", "1", "--out", js)[0] == 0
    assert run("eval", "--expr", "bsh,tsh->bth|h", "--shapes", "[[2,3,9],[4,3,3]]", "--seed", "1", "--out", bn)[0] == 0
    a = wire.tensor_from_json(open(js).read())
    b = wire.tensor_from_binary(open(bn, "rb").read())
    assert a.shape == (2, 4, 9) and np.array_equal(a, b)
    from oracle import np_oracle as npo
    x = npo.fill_random([2, 3, 9], 1).astype(np.float32).astype(np.float64)
    w = npo.fill_random([4, 3, 3], 2).astype(np.float32).astype(np.float64)
    ref, _ = npo.execute("bsh,tsh->bth|h", [[2, 3, 9], [4, 3, 3]], [(0, 1, "bth")], [x, w])
    assert np.abs(a - ref).max() / np.abs(ref).max() < 1e-5


@pytest.mark.gpu
def test_eval_mismatch_exit_code():
    # a tolerance no FP32 reassociation meets forces the numerical-mismatch code
    desc = '{"kind":"CP","T":[8],"S":[6],"H":3,"W":3,"Hp":10,"Wp":10,"B":2,"rank":5}'
    rc, out, _ = run("eval", "--layer", desc, "--seed", "3", "--plan", "both", "--tol", "0")
    assert rc in (0, 4)
    if "deviation 0.000e+00" not in out:
        assert rc == 4
