"""merge_like_modes / unmerge_modes (kernels.hpp:88-98, kernels.cpp:186-286), the reference's
public like-mode merging, against the compiled reference: the device permute
must reproduce the reference's data bit-for-bit (a pure permutation), the merged subscripts,
dims and MergeRecord exactly, and unmerge must restore the member axes."""
import numpy as np
import pytest

import paper_2401_03384_b200 as ce
from oracle import np_oracle as npo

CASES = [
    # one-input expressions whose classify() gives the classes of the merged operand's atoms
    ("abcd,cb->ad", [3, 4, 5, 2]),                    # batch / contraction / free mix
    ("bs(r1)hw,(r1)thw->bthw|hw", [2, 3, 4, 5, 6]),    # conv atoms h, w stay unmerged
    ("bshw,tshw->bthw|hw", [2, 3, 5, 6]),
    ("ijkl,kl->ij", [2, 3, 4, 5]),
    ("x(ab)y,y->x(ab)", [3, 4, 5]),
]


def _first_input(expr):
    return expr.split("->")[0].split(",")[0]


@pytest.mark.gpu
@pytest.mark.parametrize("expr,dims", CASES)
def test_merge_like_modes_matches_reference(ctx, ref, expr, dims):
    import torch
    from paper_2401_03384_b200.device import merge_like_modes, unmerge_modes
    data = npo.fill_random(dims, 17).astype(np.float32)
    r_data, r_subs, r_dims, r_rec, r_usubs, r_udims = ref.merge_like_modes(expr, dims, data.astype(np.float64))
    classes = ce.classify(expr)
    t = torch.tensor(data, device="cuda:0")
    m, msubs, rec = merge_like_modes(ctx, t, _first_input(expr), classes)
    torch.cuda.synchronize()
    assert msubs == r_subs and list(m.shape) == r_dims and rec == r_rec
    assert np.array_equal(m.cpu().numpy().astype(np.float64), r_data)
    u, usubs = unmerge_modes(m, msubs, rec)
    assert usubs == r_usubs and list(u.shape) == r_udims


def test_unmerge_modes_host_only():
    from paper_2401_03384_b200._lib import check, lib
    import ctypes
    d = (ctypes.c_int64 * 3)(6, 20, 7)
    us = ctypes.create_string_buffer(256)
    ud = (ctypes.c_int64 * 16)()
    ur = ctypes.c_int()
    check(lib().ce_unmerge_modes(b"(ab)(cd)e", d, b"ab=a:2,b:3;cd=c:4,d:5", us, len(us), ud, ctypes.byref(ur)))
    assert us.value.decode() == "abcde" and list(ud[:ur.value]) == [2, 3, 4, 5, 7]
    with pytest.raises(ce.CeError):
        check(lib().ce_unmerge_modes(b"(ab)e", (ctypes.c_int64 * 2)(7, 7), b"ab=a:2,b:3", us, len(us), ud,
                                     ctypes.byref(ur)))
