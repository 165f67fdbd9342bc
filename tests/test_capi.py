"""The C-ABI library loads and exports every symbol include/ce/ce.h declares (no GPU needed)."""
import ctypes
import os
import re

from paper_2401_03384_b200 import _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "ce", "ce.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ce_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_bindings_cover_header():
    assert set(declared_functions()) == set(_lib.SIGNATURES)


def test_version_and_error_path():
    lib = _lib.lib()
    assert b"sm_100a" in lib.ce_version()
    import paper_2401_03384_b200 as ce
    try:
        ce.parse("ab->a->b")
    except ce.ParseError as e:
        assert e.code == 2 and "duplicate" in str(e)
    else:
        raise AssertionError("expected ParseError")
